"""Motion-detection actor over the C ABI (test/bench harness view)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DF_MOTION_GRAY, DF_MOTION_RGB, call, lib, require_gpu
from .device import Buffer, Stream

GRAY, RGB = DF_MOTION_GRAY, DF_MOTION_RGB


class MotionActor:
    """Fused gray/gauss/thres/median actor with its delay token in HBM."""

    def __init__(self, width: int, height: int, fmt: int = GRAY, threshold: int = 32, device: int = 0):
        require_gpu()
        self.width, self.height, self.fmt, self.threshold = int(width), int(height), int(fmt), int(threshold)
        self.device = device
        h = C.c_void_p()
        call("df_motion_create", device, self.width, self.height, self.fmt, self.threshold, C.byref(h))
        self.handle = h

    @property
    def in_frame_bytes(self) -> int:
        return self.width * self.height * self.fmt

    @property
    def out_frame_bytes(self) -> int:
        return self.width * self.height

    def set_prev_frame(self, frame: Buffer | None, stream: Stream | None = None, offset: int = 0):
        call("df_motion_set_prev_frame", self.handle, frame.at(offset) if frame is not None else None,
             stream.handle if stream else None)

    def fire(self, inp: Buffer, out: Buffer, frames: int, stream: Stream | None = None,
             in_offset: int = 0, out_offset: int = 0):
        call("df_motion_fire", self.handle, inp.at(in_offset), out.at(out_offset), int(frames),
             stream.handle if stream else None)

    def fire_halo(self, halo: Buffer, inp: Buffer, out: Buffer, frames: int, stream: Stream | None = None,
                  halo_offset: int = 0, in_offset: int = 0, out_offset: int = 0):
        """Shard firing: `halo` (the previous shard's last input frame) stands
        in for the delay token; gauss(halo) is computed inside the firing."""
        call("df_motion_fire_halo", self.handle, halo.at(halo_offset), inp.at(in_offset), out.at(out_offset),
             int(frames), stream.handle if stream else None)

    @property
    def kernel_name(self) -> str:
        """The kernel a firing launches (for 16-byte aligned inputs)."""
        return lib().df_motion_kernel_name(self.handle).decode()

    def fire_channels(self, in_ch, delay_ch, out_ch, stream: Stream | None = None):
        call("df_motion_fire_channels", self.handle, in_ch.handle, delay_ch.handle, out_ch.handle,
             stream.handle if stream else None)

    def run_host(self, inp: np.ndarray, out: np.ndarray, chunk_frames: int = 0, stream: Stream | None = None):
        assert inp.dtype == np.uint8 and out.dtype == np.uint8
        frames = inp.size // self.in_frame_bytes
        assert out.size >= frames * self.out_frame_bytes
        call("df_motion_run_host", self.handle, inp.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
             frames, int(chunk_frames), stream.handle if stream else None)

    def close(self):
        if self.handle:
            lib().df_motion_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(frames: np.ndarray, width: int, height: int, threshold: int = 32, fmt: int = GRAY,
        device: int = 0) -> np.ndarray:
    """GPU equivalent of oracle_motion_detection_raw (proj/src/motion.cpp:236-252)."""
    frames = np.ascontiguousarray(frames, np.uint8).reshape(-1)
    a = MotionActor(width, height, fmt, threshold, device)
    out = np.empty(frames.size // fmt, np.uint8)
    a.run_host(frames, out)
    a.close()
    return out


def _stage(name, *args):
    call(name, *args)


def gauss5x5(img: np.ndarray, w: int, h: int) -> np.ndarray:
    src, dst = Buffer.from_array(img), Buffer(w * h)
    call("df_motion_gauss5x5", src.ptr, dst.ptr, w, h, None)
    return dst.download(np.uint8, w * h)


def median5(img: np.ndarray, w: int, h: int) -> np.ndarray:
    src, dst = Buffer.from_array(img), Buffer(w * h)
    call("df_motion_median5", src.ptr, dst.ptr, w, h, None)
    return dst.download(np.uint8, w * h)


def thres_diff(prev: np.ndarray, cur: np.ndarray, w: int, h: int, thr: int) -> np.ndarray:
    p, c, o = Buffer.from_array(prev), Buffer.from_array(cur), Buffer(w * h)
    call("df_motion_thres_diff", p.ptr, c.ptr, o.ptr, w, h, thr, None)
    return o.download(np.uint8, w * h)


def rgb_to_gray(rgb: np.ndarray) -> np.ndarray:
    n = rgb.size // 3
    src, dst = Buffer.from_array(rgb), Buffer(n)
    call("df_motion_rgb_to_gray", src.ptr, dst.ptr, n, None)
    return dst.download(np.uint8, n)
