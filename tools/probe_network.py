"""Probe: where the on-device network's per-step overhead over the bare
motion firing goes -- bare firing (graph / stream launches), channel-bound
firing alone (delay channel only commits on device), + source/sink commits."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_1611_03226_b200 import _lib, device, motion
from paper_1611_03226_b200.channel import DeviceChannel

p = bench.WORKLOADS["motion720"][1]
W, H, F, fmt = p["w"], p["h"], p["frames"], p["fmt"]
s = device.Stream()
cin = DeviceChannel(W * H * fmt, F)
cout = DeviceChannel(W * H, F)
delay = DeviceChannel(W * H, 1, has_delay=True, initial_token=np.zeros(W * H, np.uint8))
L = _lib.lib()
_lib.call("df_fill_random_u8", C.c_void_p(L.df_channel_storage(cin.handle)), cin.capacity_bytes, 77, s.handle)
a = motion.MotionActor(W, H, fmt, 32)
inp = device.Buffer(F * W * H * fmt)
out = device.Buffer(F * W * H)
_lib.call("df_fill_random_u8", inp.ptr, inp.nbytes, 5, s.handle)


def bare():
    a.fire(inp, out, F, s)


def network():
    wr = cin.write_start(F)
    cin.write_end(wr, s)
    a.fire_channels(cin, delay, cout, s)
    rd = cout.read_start(F)
    cout.read_end(rd, s)


def commits_only():
    wr = cin.write_start(F)
    cin.write_end(wr, s)
    rd = cin.read_start(F)  # (host reader here: commits only, no firing)
    cin.read_end(rd, s)


def channel_firing_only():  # timing only: without the endpoint commits the channel state is violated
    a.fire_channels(cin, delay, cout, s)


for name, fn in (("bare firing, stream launches", bare), ("network step", network),
                 ("channel-bound firing alone (state violated; timing only)", channel_firing_only)):
    print(f"{name}: {bench._timed_steps(fn, 20, 5, s) * 1e3:.1f} us")
cin2 = DeviceChannel(16, 4)
def two_commits():
    wr = cin2.write_start(4)
    cin2.write_end(wr, s)
    rd = cin2.read_start(4)
    cin2.read_end(rd, s)
print(f"two host-endpoint commits alone: {bench._timed_steps(two_commits, 50, 5, s) * 1e3:.1f} us")
