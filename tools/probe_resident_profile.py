import sys, os
sys.path.insert(0, os.getcwd())
from oracle import oracle as O
from paper_1611_03226_b200 import host_api as H
f = O.synth_bytes(300 * 1280 * 720, 5)
for ctas in (32, 64, 96):
    out, ms, fir = H.motion_run_resident(f, 1280, 720, 32, rate=1, ctas=ctas)
    print(f"ctas={ctas}: {300 / (ms / 1e3):.0f} fps", flush=True)
x = O.synth_samples(1 << 20, 810)
taps = O.random_taps(808)
y, ms, fir, _ = H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=16)
print(f"dpd1 {2**20 / (ms / 1e3) / 1e6:.0f} Msps", flush=True)
