"""Resident DPD-1 at several CTA counts per branch, checked against the
oracle (run from the repo root)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from paper_1611_03226_b200 import host_api as H
x = O.synth_samples(1 << 20, 810)
taps = O.random_taps(808)
want = O.dpd(x, taps, [3], 65536)
for bc in (16, 24, 32, 36):
    try:
        H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=bc)
        ms = [H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=bc)[1] for _ in range(3)]
        y = H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=bc)[0]
        print(f"branch_ctas={bc}: {2**20 / (np.median(ms) / 1e3) / 1e6:.0f} Msps exact={np.array_equal(y.view(np.uint32), want.view(np.uint32))}", flush=True)
    except Exception as e:
        print(bc, "error", e)
