"""Probe: zero-copy DPD firing -- the kernel reads its input from and
writes its output to pinned host memory directly (UVA), vs the staged
df_dpd_run_host.  Also checks the result against the staged run."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1611_03226_b200 import _lib, device, dpd


def t(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e6


for name, N, period, T, sched in (("dpd1", 1 << 20, 65536, 10, [3]), ("dpd3", 1 << 26, 4096, 10, [(1 << (1 + i % 10)) - 1 for i in range(10)]),
                                  ("dpd5", 1 << 27, 65536, 32, [0x3FF])):
    taps = np.random.default_rng(808).uniform(-0.5, 0.5, (10, 10, 2)).astype(np.float32) if T == 10 else np.random.default_rng(1).uniform(-0.5, 0.5, (10, T, 2)).astype(np.float32)
    actor = dpd.DpdActor(period, taps)
    hin = device.PinnedArray(2 * N, np.float32)
    hout = device.PinnedArray(2 * N, np.float32)
    hin.array[:] = np.random.default_rng(0).uniform(-1, 1, 2 * N).astype(np.float32)
    K = N // period
    ctrl = device.Buffer(4 * K)
    dpd.config_tokens(np.array(sched, np.uint16), 0, K, ctrl)
    lib = _lib.lib()

    def zc():
        actor.reset()
        _lib.call("df_dpd_fire", actor.handle, ctrl.ptr, hin.ptr, hout.ptr, K, None)
        _lib.call("df_stream_synchronize", None)

    def staged():
        actor.reset()
        actor.run_host(hin.array, hout.array, np.array(sched, np.uint16))

    us_s = t(staged, 5)
    ref = hout.array.copy()
    us_z = t(zc, 5)
    same = np.array_equal(ref.view(np.uint32), hout.array.view(np.uint32))
    print(f"{name}: staged {us_s:.1f} us ({N / us_s:.0f} Msps), zero-copy {us_z:.1f} us ({N / us_z:.0f} Msps), identical={same}")
    actor.close()
    hin.free()
    hout.free()
