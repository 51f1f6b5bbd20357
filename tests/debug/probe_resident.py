"""Probe: the reference-shaped networks as device-resident actors (one
persistent kernel; dfh_*_run_resident) -- sink-active throughput (the
reference's metric) and wall time, at BASELINE sizes, for a few CTA counts,
checked against the oracle (so it lives with the tests, not under tools/)."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
from oracle import oracle as O  # noqa: E402
from paper_1611_03226_b200 import host_api as H  # noqa: E402

x = O.synth_samples(1 << 20, 810)
taps = O.random_taps(808)
for ctas in (4, 8, 16):
    H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=ctas)
    t = time.perf_counter()
    y, ms, fir, _ = H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=ctas)
    wall = time.perf_counter() - t
    print(f"dpd1 resident branch_ctas={ctas}: sink-active {2**20 / (ms / 1e3) / 1e6:.0f} Msps, "
          f"wall {2**20 / wall / 1e6:.0f} Msps, exact={np.array_equal(y, O.dpd(x, taps, [3], 65536))}", flush=True)
x3 = O.synth_samples(1 << 22, 5)
ramp = np.array([(1 << (1 + i % 10)) - 1 for i in range(10)], np.uint16)
for ctas in (4, 8):
    t = time.perf_counter()
    y, ms, fir, _ = H.dpd_run_resident(x3, taps, ramp, 4096, allow_single_branch=True, branch_ctas=ctas)
    wall = time.perf_counter() - t
    print(f"dpd3 (2^22) resident branch_ctas={ctas}: sink-active {2**22 / (ms / 1e3) / 1e6:.0f} Msps, "
          f"wall {2**22 / wall / 1e6:.0f} Msps", flush=True)
f = O.synth_bytes(300 * 1280 * 720, 5)
for ctas in (16, 64):
    t = time.perf_counter()
    out, ms, fir = H.motion_run_resident(f, 1280, 720, 32, rate=1, ctas=ctas)
    wall = time.perf_counter() - t
    print(f"motion720 gray x300 resident ctas={ctas}: sink-active {300 / (ms / 1e3):.0f} fps, wall {300 / wall:.0f} fps",
          flush=True)
