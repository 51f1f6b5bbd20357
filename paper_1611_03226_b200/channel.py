"""Device channel over the C ABI, mirroring dynflow::Channel
(proj/include/dynflow/channel.hpp:71-135)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DfChanStats, DfRegion, call, lib, require_gpu
from .device import Stream


def capacity_tokens(rate: int, has_delay: bool) -> int:
    return int(lib().df_slot_capacity(rate, int(has_delay)))


def write_slot(rate: int, has_delay: bool, phase: int) -> int:
    return int(lib().df_slot_write_first(rate, int(has_delay), phase))


def read_slot(rate: int, has_delay: bool, phase: int) -> int:
    return int(lib().df_slot_read_first(rate, int(has_delay), phase))


class DeviceChannel:
    def __init__(self, token_size: int, token_rate: int = 1, has_delay: bool = False,
                 initial_token: np.ndarray | None = None, device: int = 0):
        require_gpu()
        h = C.c_void_p()
        init = None
        if initial_token is not None:
            initial_token = np.ascontiguousarray(initial_token, np.uint8)
            init = initial_token.ctypes.data_as(C.c_void_p)
        call("df_channel_create", device, int(token_size), int(token_rate), int(has_delay), init, C.byref(h))
        self.handle = h
        self.token_size, self.rate, self.has_delay = int(token_size), int(token_rate), bool(has_delay)

    @property
    def capacity_tokens(self) -> int:
        return int(lib().df_channel_capacity_tokens(self.handle))

    @property
    def capacity_bytes(self) -> int:
        return int(lib().df_channel_capacity_bytes(self.handle))

    def write_start(self, n: int) -> DfRegion:
        r = DfRegion()
        call("df_channel_write_start", self.handle, n, C.byref(r))
        return r

    def write_end(self, r: DfRegion, stream: Stream | None = None):
        call("df_channel_write_end", self.handle, C.byref(r), stream.handle if stream else None)

    def read_start(self, n: int) -> DfRegion:
        r = DfRegion()
        call("df_channel_read_start", self.handle, n, C.byref(r))
        return r

    def read_end(self, r: DfRegion, stream: Stream | None = None):
        call("df_channel_read_end", self.handle, C.byref(r), stream.handle if stream else None)

    def close_stream(self, stream: Stream | None = None):
        call("df_channel_close", self.handle, stream.handle if stream else None)

    def stats(self) -> DfChanStats:
        s = DfChanStats()
        call("df_channel_stats", self.handle, C.byref(s))
        return s

    def check(self):
        call("df_channel_check", self.handle)

    def test_produce(self, first_index: int, firings: int, seed: int, stream: Stream | None = None):
        call("df_channel_test_produce", self.handle, first_index, firings, seed, stream.handle if stream else None)

    def test_consume(self, first_pos: int, firings: int, seed: int, skip_initial: bool, bad_dev,
                     stream: Stream | None = None):
        call("df_channel_test_consume", self.handle, first_pos, firings, seed, int(skip_initial), bad_dev,
             stream.handle if stream else None)

    def close(self):
        if self.handle:
            lib().df_channel_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
