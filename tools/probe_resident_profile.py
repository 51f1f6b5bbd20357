"""Per-actor leader time split (wait / fire / commit, DF_NET_PROFILE) of the
reference-shaped networks run as device-resident actors (dfh_*_run_resident):
motion 720p gray x300 at a few CTA counts per actor, DPD-1 at 16 and 32 CTAs
per branch.  Run with DF_NET_PROFILE=1 to get the split on stderr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_03226_b200 import host_api as H  # noqa: E402

f = H.synth("frames", 300 * 1280 * 720, 5)
for ctas in (32, 64, 96):
    out, ms, fir = H.motion_run_resident(f, 1280, 720, 32, rate=1, ctas=ctas)
    print(f"motion ctas={ctas}: {300 / (ms / 1e3):.0f} fps", flush=True)
x = H.synth("samples", 1 << 20, 810)
taps = H.synth("taps", 10, 808).reshape(10, 10, 2)
for bc in (16, 32):
    y, ms, fir, _ = H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=bc)
    print(f"dpd1 branch_ctas={bc}: {2**20 / (ms / 1e3) / 1e6:.0f} Msps", flush=True)
