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
