"""ctypes binding of libdf_host.so (include/df_host.h): the C++ GPU-actor
runtime running the reference's two networks end to end from host buffers."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

HOST_LIB_PATH = os.path.join(_lib.HERE, "libdf_host.so")
_h = None


class HostRunError(RuntimeError):
    pass


def lib():
    global _h
    if _h is None:
        _lib.lib()  # libdf_cuda.so first (libdf_host.so links it via $ORIGIN)
        if not os.path.exists(HOST_LIB_PATH):
            raise RuntimeError(f"{HOST_LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(HOST_LIB_PATH)
        L.dfh_last_error.restype = C.c_char_p
        L.dfh_dpd_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                  C.c_void_p, C.c_size_t, C.c_uint32, C.c_int, C.POINTER(C.c_double),
                                  C.POINTER(C.c_uint64)]
        L.dfh_motion_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint, C.c_uint, C.c_int,
                                     C.c_uint8, C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.dfh_motion_run_mixed.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint, C.c_uint,
                                           C.c_uint8, C.c_uint32, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
        L.dfh_validate_demo.argtypes = [C.c_int]
        L.dfh_dpd_run_resident.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, C.c_double,
                                           C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
        L.dfh_motion_run_resident.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint, C.c_uint,
                                              C.c_uint8, C.c_uint32, C.c_uint32, C.c_double,
                                              C.POINTER(C.c_double), C.c_void_p]
        L.dfh_delay_chain_run.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_uint64, C.c_void_p]
        L.dfh_memory.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_uint32, C.c_uint32, C.c_int,
                                 C.POINTER(C.c_uint64)]
        L.dfh_parse_schedule.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.dfh_parse_taps.argtypes = [C.c_char_p, C.c_uint32, C.c_void_p]
        L.dfh_read_pgm.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint), C.POINTER(C.c_uint),
                                   C.POINTER(C.c_uint64)]
        L.dfh_write_pgm.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.c_uint, C.c_uint]
        L.dfh_read_raw_frames.argtypes = [C.c_char_p, C.c_uint, C.c_uint, C.c_int, C.c_void_p, C.c_size_t,
                                          C.POINTER(C.c_uint64)]
        L.dfh_read_cf32.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]
        L.dfh_write_file.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t]
        L.dfh_bulk_kernel_run.argtypes = [C.c_int, C.c_uint32, C.c_uint64, C.c_int, C.c_void_p]
        L.dfh_channel_class_demo.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_uint32, C.c_void_p,
                                             C.POINTER(C.c_int)]
        L.dfh_synth.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
        L.dfh_encode_config.argtypes = [C.c_uint16, C.c_void_p]
        L.dfh_decode_config.argtypes = [C.c_void_p, C.POINTER(C.c_uint16)]
        L.dfh_dynamic_cpu_run.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_void_p]
        _h = L
    return _h


def _check(rc):
    if rc != 0:
        raise HostRunError(f"[{rc}] {lib().dfh_last_error().decode(errors='replace')}")


def dpd_run(inp: np.ndarray, taps: np.ndarray, schedule, period: int, batch: int = 1, device: int = 0,
            out: np.ndarray | None = None, allow_single_branch: bool = False):
    """run(dpd::build_network(params)) on the GPU; returns (output, sink_active_ms, dpd_firings).
    Masks must have 2..10 active branches (the reference's check_config), or
    1..10 with allow_single_branch (extension)."""
    inp = np.ascontiguousarray(inp, np.float32).reshape(-1)
    taps = np.ascontiguousarray(taps, np.float32)
    T = taps.shape[1]
    sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    out = np.empty_like(inp) if out is None else out
    ms, fir = C.c_double(0), C.c_uint64(0)
    _check(lib().dfh_dpd_run(device, inp.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), inp.size // 2,
                             period, T, taps.ctypes.data_as(C.c_void_p), sched.ctypes.data_as(C.c_void_p),
                             sched.size, batch, int(allow_single_branch), C.byref(ms), C.byref(fir)))
    return out, ms.value, fir.value


def motion_run(frames: np.ndarray, width: int, height: int, fmt: int = 1, threshold: int = 32, rate: int = 1,
               device: int = 0, out: np.ndarray | None = None):
    """run(motion::build_network(params)) on the GPU; returns (masks, sink_active_ms, delay_tokens_written)."""
    frames = np.ascontiguousarray(frames, np.uint8).reshape(-1)
    n = frames.size // (width * height * fmt)
    out = np.empty(n * width * height, np.uint8) if out is None else out
    ms, dw = C.c_double(0), C.c_uint64(0)
    _check(lib().dfh_motion_run(device, frames.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), n, width,
                                height, fmt, threshold, rate, C.byref(ms), C.byref(dw)))
    return out, ms.value, dw.value


def motion_run_mixed(rgb: np.ndarray, width: int, height: int, threshold: int = 32, rate: int = 1,
                     device: int = 0, fail_at_firing: int = -1):
    """run(motion::build_mixed_network(params)): CPU gray + census actors around the
    GPU motion actor; returns (masks, per-frame moving-pixel counts, sink_active_ms)."""
    rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
    n = rgb.size // (width * height * 3)
    out = np.empty(n * width * height, np.uint8)
    counts = np.zeros(n, np.uint32)
    ms = C.c_double(0)
    _check(lib().dfh_motion_run_mixed(device, rgb.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), n,
                                      width, height, threshold, rate, counts.ctypes.data_as(C.c_void_p),
                                      fail_at_firing, C.byref(ms)))
    return out, counts, ms.value


def memory(app: str, shape: str, width: int = 320, height: int = 240, rate: int = 1, period: int = 65536):
    """(channel count, Eq. 1 buffer bytes) of a network shape -- cmd_mem.
    app: 'motion' | 'dpd'; shape: 'b200' (this library's network) | 'reference'."""
    tot = C.c_uint64(0)
    n = lib().dfh_memory(0 if app == "motion" else 1, width, height, rate, period,
                         0 if shape == "b200" else 1, C.byref(tot))
    if n < 0:
        raise HostRunError(lib().dfh_last_error().decode(errors="replace"))
    return n, tot.value


def validate_demo(which: int) -> int:
    return int(lib().dfh_validate_demo(which))


def delay_chain_run(rate: int, sink_first: bool, firings: int, device: int = 0) -> np.ndarray:
    """source -> sink over one delay channel (dfh_delay_chain_run); returns
    the sink's tokens as uint64 (initial token 2^64-1, then 1, 2, ...)."""
    out = np.zeros(firings * rate, np.uint64)
    _check(lib().dfh_delay_chain_run(device, rate, int(sink_first), firings, out.ctypes.data_as(C.c_void_p)))
    return out


DPD_ACTORS = ["source", "config", "split"] + [f"branch{b:02d}" for b in range(1, 11)] + ["adder", "sink"]
MOTION_ACTORS = ["source", "gauss", "thres", "med", "sink"]


def dpd_run_resident(inp: np.ndarray, taps: np.ndarray, schedule, period: int, device: int = 0,
                     allow_single_branch: bool = False, branch_ctas: int = 16, timeout_s: float = 30.0):
    """The reference's 15-actor DPD network as device-resident actors (one
    persistent kernel); returns (output, sink_active_ms, {actor: firings},
    channel tokens written [56])."""
    inp = np.ascontiguousarray(inp, np.float32).reshape(-1)
    taps = np.ascontiguousarray(taps, np.float32)
    T = taps.shape[1]
    sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    out = np.empty_like(inp)
    ms = C.c_double(0)
    fir = np.zeros(len(DPD_ACTORS), np.uint64)
    tok = np.zeros(56, np.uint64)
    _check(lib().dfh_dpd_run_resident(device, inp.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                      inp.size // 2, period, T, taps.ctypes.data_as(C.c_void_p),
                                      sched.ctypes.data_as(C.c_void_p), sched.size, int(allow_single_branch),
                                      branch_ctas, timeout_s, C.byref(ms), fir.ctypes.data_as(C.c_void_p),
                                      tok.ctypes.data_as(C.c_void_p)))
    return out, ms.value, dict(zip(DPD_ACTORS, fir.tolist())), tok


def motion_run_resident(frames: np.ndarray, width: int, height: int, threshold: int = 32, rate: int = 1,
                        device: int = 0, ctas: int = 64, timeout_s: float = 30.0):
    """The reference's 5-actor motion network (gauss_thres_prev delay channel)
    as device-resident actors; returns (masks, sink_active_ms, {actor: firings})."""
    frames = np.ascontiguousarray(frames, np.uint8).reshape(-1)
    n = frames.size // (width * height)
    out = np.empty(n * width * height, np.uint8)
    ms = C.c_double(0)
    fir = np.zeros(5, np.uint64)
    _check(lib().dfh_motion_run_resident(device, frames.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                         n, width, height, threshold, rate, ctas, timeout_s, C.byref(ms),
                                         fir.ctypes.data_as(C.c_void_p)))
    return out, ms.value, dict(zip(MOTION_ACTORS, fir.tolist()))


# ---- data formats (include/df_host.h, df/io.hpp; proj/src/bench.cpp, dpd.cpp:393-462) ----
def parse_schedule(text: str) -> np.ndarray:
    """The reference's schedule text format -> one 10-bit mask per entry (uint16)."""
    n = C.c_size_t()
    b = text.encode()
    _check(lib().dfh_parse_schedule(b, None, 0, C.byref(n)))
    out = np.empty(n.value, np.uint16)
    _check(lib().dfh_parse_schedule(b, out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
    return out


def parse_taps(text: str, taps_per_branch: int = 10) -> np.ndarray:
    """The reference's taps text format -> (10, T, 2) float32 (branch-major re, im)."""
    out = np.empty((10, taps_per_branch, 2), np.float32)
    _check(lib().dfh_parse_taps(text.encode(), taps_per_branch, out.ctypes.data_as(C.c_void_p)))
    return out


def read_pgm(path: str):
    """Concatenated binary PGM (P5) frames -> (pixels uint8 [frames, h, w], width, height)."""
    w, h, f = C.c_uint(), C.c_uint(), C.c_uint64()
    p = os.fsencode(path)
    _check(lib().dfh_read_pgm(p, None, 0, C.byref(w), C.byref(h), C.byref(f)))
    px = np.empty((f.value, h.value, w.value), np.uint8)
    _check(lib().dfh_read_pgm(p, px.ctypes.data_as(C.c_void_p), px.nbytes, C.byref(w), C.byref(h), C.byref(f)))
    return px, w.value, h.value


def write_pgm(path: str, frames: np.ndarray, width: int, height: int):
    frames = np.ascontiguousarray(frames, np.uint8)
    n = frames.size // (width * height)
    _check(lib().dfh_write_pgm(os.fsencode(path), frames.ctypes.data_as(C.c_void_p), n, width, height))


def read_raw_frames(path: str, width: int, height: int, fmt: int = 1) -> np.ndarray:
    f = C.c_uint64()
    p = os.fsencode(path)
    _check(lib().dfh_read_raw_frames(p, width, height, fmt, None, 0, C.byref(f)))
    px = np.empty(f.value * width * height * fmt, np.uint8)
    _check(lib().dfh_read_raw_frames(p, width, height, fmt, px.ctypes.data_as(C.c_void_p), px.nbytes, C.byref(f)))
    return px


def read_cf32(path: str) -> np.ndarray:
    """Interleaved complex-f32 file -> float32 [2 * samples]."""
    n = C.c_uint64()
    p = os.fsencode(path)
    _check(lib().dfh_read_cf32(p, None, 0, C.byref(n)))
    out = np.empty(2 * n.value, np.float32)
    _check(lib().dfh_read_cf32(p, out.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
    return out


def write_file(path: str, data: np.ndarray):
    data = np.ascontiguousarray(data)
    _check(lib().dfh_write_file(os.fsencode(path), data.ctypes.data_as(C.c_void_p), data.nbytes))


def dynamic_cpu_run(masks, rate: int, firings: int, device: int = 0) -> np.ndarray:
    """The dynamic DPD network shape as CPU actors (dfh_dynamic_cpu_run): int32 [firings * rate]."""
    m = np.ascontiguousarray(masks, np.uint32)
    out = np.empty(firings * rate, np.int32)
    _check(lib().dfh_dynamic_cpu_run(device, m.ctypes.data_as(C.c_void_p), m.size, rate, firings,
                                     out.ctypes.data_as(C.c_void_p)))
    return out


def encode_config(mask: int) -> bytes:
    out = (C.c_uint8 * 4)()
    _check(lib().dfh_encode_config(mask, out))
    return bytes(out)


def decode_config(b: bytes) -> int:
    buf = (C.c_uint8 * 4).from_buffer_copy(b[:4])
    m = C.c_uint16()
    _check(lib().dfh_decode_config(buf, C.byref(m)))
    return m.value


def synth(what: str, n: int, seed: int) -> np.ndarray:
    """The library's copies of the reference's generators (dfh_synth)."""
    kind, dtype, count = {"schedule": (0, np.uint16, n), "taps": (1, np.float32, 20 * n),
                          "samples": (2, np.float32, 2 * n), "frames": (3, np.uint8, n)}[what]
    out = np.empty(count, dtype)
    _check(lib().dfh_synth(kind, n, seed, out.ctypes.data_as(C.c_void_p)))
    return out


def bulk_kernel_run(rate: int, firings: int, bad: bool = False, device: int = 0) -> np.ndarray:
    out = np.empty(firings * rate, np.int32)
    _check(lib().dfh_bulk_kernel_run(device, rate, firings, int(bad), out.ctypes.data_as(C.c_void_p)))
    return out


def channel_class_demo(rate: int, delay: bool, firings: int, device: int = 0):
    out = np.empty(firings * rate, np.uint32)
    st = C.c_int()
    _check(lib().dfh_channel_class_demo(device, rate, int(delay), firings, out.ctypes.data_as(C.c_void_p),
                                        C.byref(st)))
    return out, st.value
