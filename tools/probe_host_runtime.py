"""Probe: the C++ network runtime's drop-in runs (dfh_motion_run /
dfh_dpd_run: build_network + run with host spans, as cmd_motion / cmd_dpd)
against the C-ABI host-buffer firing (df_*_run_host) on the bench configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1611_03226_b200 import device, dpd, host_api, motion

W, H, F = 1280, 720, 300
rgb = device.PinnedArray(F * W * H * 3, np.uint8)
rgb.array[:] = np.random.default_rng(1).integers(0, 256, F * W * H * 3, dtype=np.uint8)
out = device.PinnedArray(F * W * H, np.uint8)
a = motion.MotionActor(W, H, motion.RGB, 32)
a.run_host(rgb.array, out.array)
t = time.perf_counter(); a.run_host(rgb.array, out.array); t_motion_pinned = t1 = time.perf_counter() - t
a2 = motion.MotionActor(W, H, motion.RGB, 32)  # fresh delay token (black), like a new network run
a2.run_host(rgb.array, out.array)
ref = out.array.copy()
mout = device.PinnedArray(F * W * H, np.uint8)
for rate in (10, 30, 60, 150, 300):
    host_api.motion_run(rgb.array, W, H, fmt=3, rate=rate, out=mout.array)
    t = time.perf_counter()
    got, sink_ms, _ = host_api.motion_run(rgb.array, W, H, fmt=3, rate=rate, out=mout.array)
    t2 = time.perf_counter() - t
    print(f"motion 720p x300: run_host {F / t1:.0f} fps; dfh_motion_run rate {rate}: wall {F / t2:.0f} fps, "
          f"sink-active {F / (sink_ms / 1e3):.0f} fps (cmd_motion's metric), identical={np.array_equal(got, ref)}")

N, period = 1 << 20, 65536
x = device.PinnedArray(2 * N, np.float32)
x.array[:] = np.random.default_rng(810).uniform(-1, 1, 2 * N).astype(np.float32)
taps = np.random.default_rng(808).uniform(-0.5, 0.5, (10, 10, 2)).astype(np.float32)
d = dpd.DpdActor(period, taps)
y = device.PinnedArray(2 * N, np.float32)
sched = np.array([3], np.uint16)
d.run_host(x.array, y.array, sched)
d.reset()
t = time.perf_counter(); d.run_host(x.array, y.array, sched); t1 = time.perf_counter() - t
for batch in (1, 4, 16):
    host_api.dpd_run(x.array, taps, sched, period, batch=batch, out=y.array)
    t = time.perf_counter()
    got, sink_ms, _ = host_api.dpd_run(x.array, taps, sched, period, batch=batch, out=y.array)
    t2 = time.perf_counter() - t
    print(f"dpd 2^20: run_host {N / t1 / 1e6:.0f} Msps; dfh_dpd_run batch {batch}: wall {N / t2 / 1e6:.0f} Msps, "
          f"sink-active {N / (sink_ms / 1e3) / 1e6:.0f} Msps (cmd_dpd's metric)")

# pageable user buffers (what cmd_motion / cmd_dpd pass: std::vector storage)
pg_in = np.array(rgb.array)
for rate in (10, 60):
    host_api.motion_run(pg_in, W, H, fmt=3, rate=rate)
    t = time.perf_counter()
    got, sink_ms, _ = host_api.motion_run(pg_in, W, H, fmt=3, rate=rate)
    t2 = time.perf_counter() - t
    print(f"pageable buffers, dfh_motion_run rate {rate}: wall {F / t2:.0f} fps, sink-active {F / (sink_ms / 1e3):.0f} fps")

# df_*_run_host with pageable caller buffers (staged through pinned slots
# with parallel host copies) vs pinned
pg_out = np.empty(F * W * H, np.uint8)
a3 = motion.MotionActor(W, H, motion.RGB, 32)
a3.run_host(pg_in, pg_out)
t = time.perf_counter(); a3.run_host(pg_in, pg_out); t3 = time.perf_counter() - t
print(f"run_host, pageable buffers: {F / t3:.0f} fps (pinned: {F / t_motion_pinned:.0f})")
pgx = np.array(x.array)
pgy = np.empty_like(pgx)
d.run_host(pgx, pgy, sched)
t = time.perf_counter(); d.run_host(pgx, pgy, sched); t4 = time.perf_counter() - t
print(f"dpd run_host, pageable buffers: {N / t4 / 1e6:.0f} Msps")
