"""Probe: DPD-1 end to end from host buffers, three ways --
(1) df_dpd_run_host (staged: H2D / fire / D2H on copy engines),
(2) hybrid: copy-engine H2D per chunk, the firing stores its output
    straight into the pinned host buffer (mapped, posted PCIe writes),
(3) as (2) with 1..8 chunks.  Checks results are identical."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1611_03226_b200 import _lib, device, dpd

N, period = 1 << 20, 65536
K = N // period
actor = dpd.DpdActor(period, np.random.default_rng(808).uniform(-0.5, 0.5, (10, 10, 2)).astype(np.float32))
hin = device.PinnedArray(2 * N, np.float32)
hout = device.PinnedArray(2 * N, np.float32)
hin.array[:] = np.random.default_rng(0).uniform(-1, 1, 2 * N).astype(np.float32)
sched = np.array([3], np.uint16)
ctrl = device.Buffer(4 * K)
dpd.config_tokens(sched, 0, K, ctrl)
din = device.Buffer(8 * N)


def t(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e6


def staged():
    actor.reset()
    actor.run_host(hin.array, hout.array, sched)


us = t(staged)
ref = hout.array.copy()
print(f"staged run_host: {us:.1f} us ({N / us:.0f} Msps)")
streams = [torch.cuda.Stream() for _ in range(2)]


def hybrid(nch):
    def run():
        actor.reset()
        torch.cuda.synchronize()
        bpc = K // nch
        evs = []
        h2d, cs = streams
        for c in range(nch):
            off = 8 * period * bpc * c
            nbytes = 8 * period * bpc
            _lib.call("df_memcpy_h2d", din.at(off), C.c_void_p(hin.ptr.value + off), nbytes, C.c_void_p(h2d.cuda_stream))
            ev = torch.cuda.Event()
            ev.record(h2d)
            cs.wait_event(ev)
            _lib.call("df_dpd_fire", actor.handle, ctrl.at(4 * bpc * c), din.at(off),
                      C.c_void_p(hout.ptr.value + off), bpc, C.c_void_p(cs.cuda_stream))
        cs.synchronize()
    return run


for nch in (1, 2, 4, 8, 16):
    us = t(hybrid(nch))
    same = np.array_equal(hout.array.view(np.uint32), ref.view(np.uint32))
    print(f"hybrid {nch} chunks: {us:.1f} us ({N / us:.0f} Msps) identical={same}")
