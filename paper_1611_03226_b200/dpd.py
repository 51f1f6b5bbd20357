"""DPD actor over the C ABI (test/bench harness view of libdf_cuda).

Mirrors the reference's DPD vocabulary (proj/include/dynflow/dpd.hpp):
ConfigToken masks (bit b-1 = branch b), taps as (10, T) complex, a period
of samples per token, schedule cycling per period.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import call, lib, require_gpu
from .device import Buffer, Stream

BRANCHES = 10


def first_n(k: int) -> int:
    """ConfigToken::first_n (proj/include/dynflow/dpd.hpp:33)."""
    return (1 << k) - 1


def check_config(mask: int, allow_single: bool = True) -> None:
    """check_config (proj/src/dpd.cpp:49-58); k = 1 allowed as an extension."""
    if mask >> BRANCHES:
        raise ValueError("config token names a branch beyond 10")
    k = bin(mask).count("1")
    lo = 1 if allow_single else 2
    if k < lo or k > BRANCHES:
        raise ValueError(f"active branch count {k} outside [{lo},10]")


def _taps_array(taps) -> np.ndarray:
    t = np.ascontiguousarray(np.asarray(taps, np.float32))
    if t.ndim == 2 and t.shape[0] == BRANCHES and np.iscomplexobj(taps):
        t = np.stack([np.real(taps), np.imag(taps)], -1).astype(np.float32)
    assert t.shape[0] == BRANCHES and t.shape[-1] == 2, "taps must be (10, T, 2) float32"
    return np.ascontiguousarray(t)


class DpdActor:
    """One GPU DPD actor: taps + per-branch FIR history resident in HBM."""

    def __init__(self, period: int, taps, device: int = 0):
        require_gpu()
        t = _taps_array(taps)
        self.T = int(t.shape[1])
        self.period = int(period)
        self.device = device
        h = C.c_void_p()
        call("df_dpd_create", device, self.period, self.T, t.ctypes.data_as(C.c_void_p), C.byref(h))
        self.handle = h

    def set_taps(self, taps, stream: Stream | None = None):
        t = _taps_array(taps)
        assert t.shape[1] == self.T
        call("df_dpd_set_taps", self.handle, t.ctypes.data_as(C.c_void_p), stream.handle if stream else None)

    @property
    def kernel_name(self) -> str:
        """Main kernel of the last firing (df_dpd_kernel_name)."""
        return lib().df_dpd_kernel_name(self.handle).decode()

    def reset(self, stream: Stream | None = None):
        call("df_dpd_reset", self.handle, stream.handle if stream else None)

    def state(self) -> np.ndarray:
        out = np.empty(BRANCHES * max(self.T - 1, 1) * 2, np.float32)
        call("df_dpd_get_state", self.handle, out.ctypes.data_as(C.c_void_p))
        return out[: BRANCHES * (self.T - 1) * 2].reshape(BRANCHES, self.T - 1, 2)

    def set_history(self, raw: Buffer, count: int, branch_mask: int = 0x3FF, stream: Stream | None = None,
                    offset: int = 0):
        """FIR-history halo: state as left by processing `count` raw samples."""
        call("df_dpd_set_history", self.handle, raw.at(offset), int(count), int(branch_mask),
             stream.handle if stream else None)

    def check(self):
        call("df_dpd_error", self.handle)

    def fire(self, ctrl: Buffer, inp: Buffer, out: Buffer, blocks: int, stream: Stream | None = None,
             ctrl_offset: int = 0, in_offset: int = 0, out_offset: int = 0):
        call("df_dpd_fire", self.handle, ctrl.at(ctrl_offset), inp.at(in_offset), out.at(out_offset),
             int(blocks), stream.handle if stream else None)

    def fire_halo(self, halo_tails, ctrl: Buffer, inp: Buffer, out: Buffer, blocks: int,
                  stream: Stream | None = None, ctrl_offset: int = 0, in_offset: int = 0, out_offset: int = 0):
        """Shard firing: halo_tails[b-1] = device address (int, local or an
        IPC peer pointer) of branch b's last T-1 raw samples before the
        shard, or None to keep the carried history."""
        arr = (C.c_void_p * 10)(*[C.c_void_p(t) if t else None for t in halo_tails])
        call("df_dpd_fire_halo", self.handle, arr, ctrl.at(ctrl_offset), inp.at(in_offset), out.at(out_offset),
             int(blocks), stream.handle if stream else None)

    def fire_channels(self, ctrl_ch, in_ch, out_ch, firings: int, stream: Stream | None = None):
        call("df_dpd_fire_channels", self.handle, ctrl_ch.handle, in_ch.handle, out_ch.handle,
             int(firings), stream.handle if stream else None)

    def run_host(self, inp: np.ndarray, out: np.ndarray, schedule, chunk_blocks: int = 0,
                 stream: Stream | None = None):
        """End to end from host buffers (interleaved complex64 as float32)."""
        sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
        assert inp.dtype == np.float32 and out.dtype == np.float32 and inp.size == out.size
        call("df_dpd_run_host", self.handle, inp.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
             inp.size // 2, sched.ctypes.data_as(C.c_void_p), sched.size, int(chunk_blocks),
             stream.handle if stream else None)

    def close(self):
        if self.handle:
            lib().df_dpd_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def config_tokens(schedule, first: int, count: int, ctrl: Buffer, device: int = 0,
                  stream: Stream | None = None, offset: int = 0):
    """Config actor (proj/src/dpd.cpp:206-221) run on device."""
    sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    call("df_dpd_config_tokens", device, sched.ctypes.data_as(C.c_void_p), sched.size, int(first), int(count),
         ctrl.at(offset), stream.handle if stream else None)


def run(inp: np.ndarray, taps, schedule, period: int, device: int = 0) -> np.ndarray:
    """GPU equivalent of oracle_dpd(input, taps, schedule, period) (proj/src/dpd.cpp:358-391)."""
    inp = np.ascontiguousarray(inp, np.float32).reshape(-1)
    if inp.size // 2 % period != 0:
        raise ValueError("sample count must be a multiple of the period")
    actor = DpdActor(period, taps, device)
    out = np.empty_like(inp)
    actor.run_host(inp, out, schedule)
    actor.check()
    actor.close()
    return out
