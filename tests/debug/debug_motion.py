"""Diff patterns of the fused motion kernel vs the oracle (GPU debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1611_03226_b200 import motion  # noqa: E402


def show(name, got, want, w, h):
    if np.array_equal(got, want):
        print(name, "OK")
        return
    d = (got != want).reshape(-1, h, w)
    fr = np.nonzero(d.any((1, 2)))[0]
    print(name, "bad bytes", d.sum(), "frames", fr[:20].tolist())
    f0 = fr[0]
    rows = np.nonzero(d[f0].any(1))[0]
    cols = np.nonzero(d[f0].any(0))[0]
    print("   frame", f0, "rows", rows[:40].tolist(), "cols", cols[:40].tolist())
    g = got.reshape(-1, h, w)[f0]
    wv = want.reshape(-1, h, w)[f0]
    r = rows[0]
    print("   row", r, "got ", g[r, :24].tolist())
    print("   row", r, "want", wv[r, :24].tolist())


CASES = [(96, 40, 6, 1), (96, 40, 6, 3), (96, 40, 1, 1), (96, 8, 1, 1), (64, 48, 2, 1),
         (16, 8, 1, 1), (16, 8, 2, 1), (320, 240, 64, 1)]
if len(sys.argv) > 1:
    CASES = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
def _main():
  for case in CASES:
      w, h, n, fmt = case[:4]
      chunk = case[4] if len(case) > 4 else 0
      src = O.synth_bytes(n * w * h * fmt, 606)
      a = motion.MotionActor(w, h, fmt, 32)
      got = np.empty(n * w * h, np.uint8)
      a.run_host(src, got, chunk_frames=chunk)
      want = O.motion_rgb(src, w, h) if fmt == 3 else O.motion_gray(src, w, h)
      show(f"{w}x{h}x{n} fmt{fmt} chunk{chunk}", got, want, w, h)


if __name__ == '__main__':
    _main()
