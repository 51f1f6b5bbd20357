"""Probe: motion 720p RGB x300 end to end (df_motion_run_host) vs the
staging chunk size (default: ~1/8 of the run, >= 4 MB)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1611_03226_b200 import device, motion

W, H, F = 1280, 720, 300
a = motion.MotionActor(W, H, motion.RGB, 32)
hin = device.PinnedArray(F * W * H * 3, np.uint8)
hout = device.PinnedArray(F * W * H, np.uint8)
hin.array[:] = 7
for chunk in (0, 75, 38, 25, 19, 10):
    a.run_host(hin.array, hout.array, chunk_frames=chunk)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        a.run_host(hin.array, hout.array, chunk_frames=chunk)
        ts.append(time.perf_counter() - t)
    s = statistics.median(ts)
    print(f"chunk_frames={chunk}: {s * 1e3:.2f} ms -> {F / s:.0f} frames/s")
