"""Device memory, streams and events over the C ABI (plumbing only)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import call, lib, require_gpu


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Stream:
    def __init__(self, device: int = 0):
        require_gpu()
        self.device = device
        h = C.c_void_p()
        call("df_stream_create", device, C.byref(h))
        self.handle = h

    def synchronize(self):
        call("df_stream_synchronize", self.handle)

    def close(self):
        if self.handle:
            call("df_stream_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Event:
    def __init__(self):
        h = C.c_void_p()
        call("df_event_create", C.byref(h))
        self.handle = h

    def record(self, stream: Stream | None):
        call("df_event_record", self.handle, stream.handle if stream else None)

    def synchronize(self):
        call("df_event_synchronize", self.handle)

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        call("df_event_elapsed_ms", self.handle, end.handle, C.byref(ms))
        return float(ms.value)

    def __del__(self):
        try:
            call("df_event_destroy", self.handle)
        except Exception:
            pass


class Buffer:
    """A device allocation; ``nbytes`` bytes on ``device``."""

    def __init__(self, nbytes: int, device: int = 0):
        require_gpu()
        self.nbytes = int(nbytes)
        self.device = device
        p = C.c_void_p()
        call("df_malloc", device, self.nbytes, C.byref(p))
        self.ptr = p

    @classmethod
    def from_array(cls, a: np.ndarray, device: int = 0, stream: Stream | None = None) -> "Buffer":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes, device)
        b.upload(a, stream)
        return b

    def upload(self, a: np.ndarray, stream: Stream | None = None, offset: int = 0):
        a = np.ascontiguousarray(a)
        assert offset + a.nbytes <= self.nbytes
        call("df_memcpy_h2d", C.c_void_p(self.ptr.value + offset), _ptr(a), a.nbytes,
             stream.handle if stream else None)
        if stream is None:
            call("df_stream_synchronize", None)
        else:
            stream.synchronize()

    def download(self, dtype, count: int | None = None, stream: Stream | None = None, offset: int = 0):
        itemsize = np.dtype(dtype).itemsize
        if count is None:
            count = (self.nbytes - offset) // itemsize
        out = np.empty(count, dtype)
        call("df_memcpy_d2h", _ptr(out), C.c_void_p(self.ptr.value + offset), out.nbytes,
             stream.handle if stream else None)
        if stream is None:
            call("df_stream_synchronize", None)
        else:
            stream.synchronize()
        return out

    def zero(self, stream: Stream | None = None):
        call("df_memset", self.ptr, 0, self.nbytes, stream.handle if stream else None)

    def at(self, offset: int) -> C.c_void_p:
        return C.c_void_p(self.ptr.value + offset)

    def as_tensor(self, dtype=np.uint8):
        """Zero-copy torch view (CUDA array interface) of the allocation;
        the Buffer must outlive it."""
        import torch
        dt = np.dtype(dtype)

        class _View:
            __cuda_array_interface__ = {"shape": (self.nbytes // dt.itemsize,), "typestr": dt.str,
                                        "data": (self.ptr.value, False), "version": 3}
        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def free(self):
        if self.ptr:
            call("df_free", self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedArray:
    """Page-locked host memory viewed as a numpy array (e2e H2D/D2H)."""

    def __init__(self, count: int, dtype):
        self.dtype = np.dtype(dtype)
        nbytes = max(1, int(count) * self.dtype.itemsize)
        p = C.c_void_p()
        call("df_host_alloc", nbytes, C.byref(p))
        self.ptr = p
        buf = (C.c_char * nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(count))

    def free(self):
        if self.ptr:
            self.array = None
            call("df_host_free", self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def kernel_launches() -> int:
    return int(lib().df_kernel_launches())
