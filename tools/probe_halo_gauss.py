"""Probe: cost of a shard's one-frame halo on ranks > 0 -- the separate
gauss pass (df_motion_set_prev_frame(halo) + df_motion_fire) vs the
in-kernel halo warm-up (df_motion_fire_halo), per firing of the bench's
frames per GPU."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1611_03226_b200 import _lib, motion


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (W, H, F) in ((1280, 720, 300), (3840, 2160, 40)):
    a = motion.MotionActor(W, H, 3, 32)
    inp = torch.randint(0, 255, (F * W * H * 3,), dtype=torch.uint8, device="cuda")
    halo = torch.randint(0, 255, (W * H * 3,), dtype=torch.uint8, device="cuda")
    out = torch.empty(F * W * H, dtype=torch.uint8, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    hp, ip, op = C.c_void_p(halo.data_ptr()), C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr())

    def black():
        _lib.call("df_motion_set_prev_frame", a.handle, None, s)
        _lib.call("df_motion_fire", a.handle, ip, op, F, s)

    def separate():
        _lib.call("df_motion_set_prev_frame", a.handle, hp, s)
        _lib.call("df_motion_fire", a.handle, ip, op, F, s)

    def inline():
        _lib.call("df_motion_fire_halo", a.handle, hp, ip, op, F, s)

    print(f"{W}x{H} x{F}: rank 0 (black token) {timed(black):.1f} us, separate halo gauss {timed(separate):.1f} us, "
          f"in-kernel halo {timed(inline):.1f} us")

# DPD: a rank > 0 firing reads its per-branch halo tails in-kernel
# (df_dpd_fire_halo; here local pointers stand in for the peer pointers).
from paper_1611_03226_b200 import dpd  # noqa: E402
import numpy as np  # noqa: E402

for name, N, period, T, sched in (("dpd1", 1 << 20, 65536, 10, [3]),
                                  ("dpd3", 1 << 26, 4096, 10, [(1 << (1 + i % 10)) - 1 for i in range(10)]),
                                  ("dpd5", 1 << 27, 65536, 32, [0x3FF])):
    taps = np.random.default_rng(808).uniform(-0.5, 0.5, size=(10, T, 2)).astype(np.float32)
    a = dpd.DpdActor(period, taps)
    K = N // period
    x = torch.rand(2 * N, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    ctrl = torch.empty(K, dtype=torch.int32, device="cuda")
    sn = np.array(sched, np.uint16)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("df_dpd_config_tokens", 0, sn.ctypes.data_as(C.c_void_p), sn.size, 0, K, C.c_void_p(ctrl.data_ptr()), s)
    tails = (C.c_void_p * 10)(*[C.c_void_p(x.data_ptr() + 8 * (period - (T - 1)))] * 10)
    xp, yp, cp = C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(ctrl.data_ptr())

    def plain():
        _lib.call("df_dpd_fire", a.handle, cp, xp, yp, K, s)

    def halo():
        _lib.call("df_dpd_fire_halo", a.handle, tails, cp, xp, yp, K, s)

    print(f"{name}: rank 0 firing {timed(plain):.1f} us, rank > 0 firing with in-kernel halo {timed(halo):.1f} us")
