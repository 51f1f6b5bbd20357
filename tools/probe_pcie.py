"""Probe: pinned H2D / D2H bandwidth with 1, 2 and 4 concurrent streams
(does splitting a chunk's copy across copy engines beat one stream?)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1611_03226_b200 import device

MB = 1 << 20
n = 512 * MB
h = device.PinnedArray(n, np.uint8)
h.array[:] = 1
th = torch.from_numpy(h.array)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(k, d2h=False):
    part = n // k
    torch.cuda.synchronize()
    a = time.perf_counter()
    for i in range(k):
        with torch.cuda.stream(streams[i]):
            if d2h:
                th[i * part:(i + 1) * part].copy_(d[i * part:(i + 1) * part], non_blocking=True)
            else:
                d[i * part:(i + 1) * part].copy_(th[i * part:(i + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - a


for d2h in (False, True):
    for k in (1, 2, 4):
        run(k, d2h)
        t = statistics.median(run(k, d2h) for _ in range(5))
        print(f"{'D2H' if d2h else 'H2D'} {k} stream(s): {n / t / 1e9:.1f} GB/s")
