"""Resident motion network (the reference's 5-actor shape, 720p gray x300)
at token rates r in {1, 2, 5, 10, 20} frames per token (the reference's
`rate` bench parameter, proj/src/bench.cpp:212) and a few CTA budgets;
byte-exact check against the r=1 run.  DF_NET_PROFILE=1 prints each actor's
wait / fire / commit split on stderr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_03226_b200 import host_api as H  # noqa: E402

f = H.synth("frames", 300 * 1280 * 720, 5)
base = None
for ctas in [int(c) for c in os.environ.get("CTAS", "96").split(",")]:
    for r in [int(c) for c in os.environ.get("RATES", "1,2,5,10,20").split(",")]:
        best = 0.0
        for _ in range(2):
            out, ms, fir = H.motion_run_resident(f, 1280, 720, 32, rate=r, ctas=ctas)
            best = max(best, 300 / (ms / 1e3))
        if base is None:
            base = out
        print(f"motion720gray resident ctas={ctas} rate={r}: {best:.0f} fps (sink-active), "
              f"equal_to_first={bool((out == base).all())}", flush=True)
