"""What does bench.py's flushed, per-step event timing add around a kernel?
Times (a) an empty kernel and (b) one DPD-1 firing between the same graph-captured
external event pair that bench_dpd_ours uses, after the same 256 MB L2 flush,
and (c) the same firing K times back to back without flushes (one event pair)."""
import ctypes as C
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_03226_b200 import _lib, dpd  # noqa: E402

dev = torch.device("cuda", 0)
N, period = 1 << 20, 65536
blocks = N // period
x = torch.empty(2 * N, dtype=torch.float32, device=dev)
y = torch.empty_like(x)
ctrl = torch.empty(blocks, dtype=torch.int32, device=dev)
sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.call("df_fill_random_pm1", C.c_void_p(x.data_ptr()), 2 * N, 99, sh)
s = np.array([3], np.uint16)
_lib.call("df_dpd_config_tokens", 0, s.ctypes.data_as(C.c_void_p), 1, 0, blocks, C.c_void_p(ctrl.data_ptr()), sh)
taps = np.random.default_rng(808).uniform(-0.5, 0.5, size=(10, 10, 2)).astype(np.float32)
actor = dpd.DpdActor(period, taps)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rflush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
tiny = torch.zeros(1, device=dev)
K = 20


def fire():
    _lib.call("df_dpd_fire", actor.handle, C.c_void_p(ctrl.data_ptr()), C.c_void_p(x.data_ptr()),
              C.c_void_p(y.data_ptr()), blocks, C.c_void_p(torch.cuda.current_stream().cuda_stream))


def noop():
    tiny.add_(0)


def graph_timed(work, read_flush=False):
    kev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
           for _ in range(K)]
    for _ in range(3):
        work()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(K):
            flush.fill_(i & 0xFF)
            if read_flush:
                rflush.sum(dtype=torch.int64)
            kev[i][0].record()
            work()
            kev[i][1].record()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in kev]
    return statistics.mean(t), statistics.median(t)


for name, work in (("empty kernel", noop), ("dpd1 firing", fire)):
    for rf in (False, True):
        m, md = graph_timed(work, rf)
        print(f"{name:14s} flush={'write+read' if rf else 'write':10s} per-step events: mean {m:6.2f} us median {md:6.2f} us")
# back to back, no flush: one event pair around K firings
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(K):
        fire()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"dpd1 firing    back-to-back (input L2-resident), graph of {K}: {e0.elapsed_time(e1) * 1e3 / K:6.2f} us per firing")
# rotating pool of 16 input/output pairs (256 MB > L2): every firing reads a
# cold input; one event pair around K back-to-back firings
R = 16
xs = [torch.empty(2 * N, dtype=torch.float32, device=dev) for _ in range(R)]
ys = [torch.empty(2 * N, dtype=torch.float32, device=dev) for _ in range(R)]
for t in xs:
    _lib.call("df_fill_random_pm1", C.c_void_p(t.data_ptr()), 2 * N, 7, sh)


def fire_i(i):
    _lib.call("df_dpd_fire", actor.handle, C.c_void_p(ctrl.data_ptr()), C.c_void_p(xs[i % R].data_ptr()),
              C.c_void_p(ys[i % R].data_ptr()), blocks, C.c_void_p(torch.cuda.current_stream().cuda_stream))


KR = 64
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(KR):
        fire_i(i)
torch.cuda.synchronize()
for rep in range(3):
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"dpd1 firing    rotating 16-buffer pool (256 MB, cold inputs), graph of {KR}: {e0.elapsed_time(e1) * 1e3 / KR:6.2f} us per firing")
