"""Resident DPD network (the reference's 15-actor shape): DPD-1 (period 65536,
2 branches) and the DPD-3 ramp (period 4096, 1..10 branches per block) at a
few CTA budgets per branch; sink-active throughput and, with
DF_NET_PROFILE=1, each actor leader's wait / fire / commit split (stderr)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_03226_b200 import host_api as H  # noqa: E402

taps = H.synth("taps", 10, 808).reshape(10, 10, 2)
x1 = H.synth("samples", 1 << 20, 810)
ramp = np.array([(1 << (1 + i % 10)) - 1 for i in range(10)], np.uint16)
x3 = H.synth("samples", 1 << int(os.environ.get("LOG2_N3", "22")), 811)
for bc in [int(c) for c in os.environ.get("BRANCH_CTAS", "8,32").split(",")]:
    for name, x, sched, period in (("dpd1", x1, [3], 65536), ("dpd3", x3, ramp, 4096)):
        best = 0.0
        for _ in range(2):
            y, ms, fir, _ = H.dpd_run_resident(x, taps, sched, period, branch_ctas=bc, allow_single_branch=True)
            best = max(best, x.size // 2 / (ms / 1e3) / 1e6)
        print(f"{name} resident branch_ctas={bc}: {best:.0f} Msamples/s (sink-active), "
              f"{period} samples per firing, {x.size // 2 // period} firings", flush=True)
