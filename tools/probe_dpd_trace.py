"""Timeline of one DPD firing from a DF_DPD_TRACE build (globaltimer stamps per
tile/granule warp: start, window loaded, end).  Usage (GPU box):
  DF_CUDA_LIB=paper_1611_03226_b200/variants/libdf_cuda_<v>.so python tools/probe_dpd_trace.py [dpd1|dpd3]
Prints the firing's span, per-warp latency split and warps in flight over time."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_03226_b200 import _lib, dpd  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "dpd1"
N, period, sched = {"dpd1": (1 << 20, 65536, [0b11]),
                    "dpd3": (1 << 26, 4096, [(1 << (1 + i % 10)) - 1 for i in range(10)])}[wl]
blocks = N // period
dev = torch.device("cuda", 0)
x = torch.empty(2 * N, dtype=torch.float32, device=dev)
y = torch.empty_like(x)
ctrl = torch.empty(blocks, dtype=torch.int32, device=dev)
sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.call("df_fill_random_pm1", C.c_void_p(x.data_ptr()), 2 * N, 99, sh)
s = np.array(sched, np.uint16)
_lib.call("df_dpd_config_tokens", 0, s.ctypes.data_as(C.c_void_p), s.size, 0, blocks, C.c_void_p(ctrl.data_ptr()), sh)
taps = np.random.default_rng(808).uniform(-0.5, 0.5, size=(10, 10, 2)).astype(np.float32)
actor = dpd.DpdActor(period, taps)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
lib = _lib.lib()
buf = (C.c_ulonglong * (8 << 15))()
rflush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
READFLUSH = os.environ.get('READFLUSH', '0') == '1'
cnt = C.c_uint()


def fire():
    _lib.call("df_dpd_fire", actor.handle, C.c_void_p(ctrl.data_ptr()), C.c_void_p(x.data_ptr()),
              C.c_void_p(y.data_ptr()), blocks, sh)


for _ in range(5):
    fire()
torch.cuda.synchronize()
spans = []
for rep in range(3):
    flush.fill_(rep)
    if READFLUSH:  # evict the flush's dirty lines before the timed firing
        rflush.sum(dtype=torch.int64)
    torch.cuda.synchronize()
    lib.df_debug_dpd_trace(None, C.byref(cnt))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fire()
    e1.record()
    torch.cuda.synchronize()
    lib.df_debug_dpd_trace(buf, C.byref(cnt))
    n = cnt.value
    a = np.frombuffer(buf, dtype=np.uint64, count=8 * n).reshape(n, 8).astype(np.int64)
    a = a[a[:, 1] != 0]  # slots written by this firing
    n = len(a)
    t0 = a[:, 1].min()
    st, ld, en, fi = a[:, 1] - t0, a[:, 2] - t0, a[:, 3] - t0, a[:, 4] - t0
    sm = (a[:, 0] >> 40) & 0xFFFF
    print(f"[{wl} rep {rep}] event {e0.elapsed_time(e1) * 1e3:.1f} us; {n} warp records; "
          f"span first start -> last end {en.max() / 1e3:.2f} us")
    print(f"  start: min 0 median {np.median(st) / 1e3:.2f} max {st.max() / 1e3:.2f} us")
    print(f"  load (start->loaded): median {np.median(ld - st) / 1e3:.2f} p90 {np.percentile(ld - st, 90) / 1e3:.2f} us")
    print(f"  fir (loaded->fir done): median {np.median(fi - ld) / 1e3:.2f} p90 {np.percentile(fi - ld, 90) / 1e3:.2f} us")
    print(f"  store (fir done->end): median {np.median(en - fi) / 1e3:.2f} p90 {np.percentile(en - fi, 90) / 1e3:.2f} us")
    late = en > np.percentile(en, 75)
    print(f"  last quarter of warps to end: start median {np.median(st[late]) / 1e3:.2f} load {np.median((ld - st)[late]) / 1e3:.2f} "
          f"fir {np.median((fi - ld)[late]) / 1e3:.2f} store {np.median((en - fi)[late]) / 1e3:.2f} us")
    print(f"  end: median {np.median(en) / 1e3:.2f} p90 {np.percentile(en, 90) / 1e3:.2f} max {en.max() / 1e3:.2f} us")
    # warps in flight over time, 0.5 us bins
    edges = np.arange(0, en.max() + 500, 500)
    inflight = [int(((st <= t) & (en > t)).sum()) for t in edges]
    print("  warps in flight per 0.5 us: " + " ".join(str(v) for v in inflight))
    per_sm_end = np.array([en[sm == k].max() for k in np.unique(sm)])
    print(f"  per-SM last end: min {per_sm_end.min() / 1e3:.2f} median {np.median(per_sm_end) / 1e3:.2f} "
          f"max {per_sm_end.max() / 1e3:.2f} us ({len(per_sm_end)} SMs)")
    spans.append(en.max())
    out = os.environ.get("TRACE_OUT")
    if out:
        np.save(f"{out}_{wl}_rep{rep}.npy", a)
