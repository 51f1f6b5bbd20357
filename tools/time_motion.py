"""Device time of one motion firing per input format / size (CUDA events,
median of reps).  Usage: python tools/time_motion.py [W H FRAMES]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1611_03226_b200 import motion
from paper_1611_03226_b200.device import Buffer, Event, Stream

W, H, F = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1280, 720, 300)
peak = 6549.4
for fmt, name in ((motion.GRAY, "gray"), (motion.RGB, "rgb")):
    a = motion.MotionActor(W, H, fmt)
    rng = np.random.default_rng(1)
    inp = Buffer.from_array(rng.integers(0, 256, W * H * fmt * F, dtype=np.uint8))
    out = Buffer(W * H * F)
    s = Stream()
    for _ in range(3):
        a.fire(inp, out, F, s)
    ts = []
    for _ in range(10):
        e0, e1 = Event(), Event()
        e0.record(s); a.fire(inp, out, F, s); e1.record(s); e1.synchronize()
        ts.append(e0.elapsed_ms(e1))
    ms = float(np.median(ts))
    gbs = (fmt + 1) * W * H * F / ms / 1e6
    print(f"{name} {W}x{H}x{F}: {ms:.4f} ms  {gbs:.0f} GB/s  frac {gbs / peak:.3f}")
    a.close()
