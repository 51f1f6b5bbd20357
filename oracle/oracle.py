"""ctypes bindings for the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs import this module, and only as the checker or
the timed CPU baseline.  The product package (``paper_1611_03226_b200``)
never imports it.

Two libraries:
  * ``port``: oracle/liboracle.so, our C restatement (oracle.c), cites the
    reference file:line per function;
  * ``ref``:  oracle/_ref/libdynflow_ref.so, the unmodified reference
    compiled from /root/reference/proj/src (+ ref_shim.cpp).  Optional:
    absent when /root/reference was not available at build time.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libdynflow_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_dp = C.POINTER(C.c_double)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class _Lib:
    def __init__(self, path):
        self.path = path
        self.lib = C.CDLL(path)


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise RuntimeError(f"{PORT_PATH} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(PORT_PATH)
        lib.orc_dpd.restype = C.c_int
        lib.orc_dpd.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint, C.c_void_p, C.c_size_t,
                                C.c_uint32, C.c_void_p]
        lib.orc_dpd_mt.restype = C.c_int
        lib.orc_dpd_mt.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint, C.c_void_p, C.c_size_t,
                                   C.c_uint32, C.c_void_p, C.c_uint]
        lib.orc_motion_mt.argtypes = [C.c_void_p, C.c_size_t, C.c_uint, C.c_uint, C.c_int, C.c_uint8, C.c_void_p,
                                      C.c_void_p, C.c_uint]
        lib.orc_compare_samples.restype = C.c_int64
        lib.orc_compare_samples.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_double, _dp]
        for name in ("orc_capacity_tokens", "orc_write_slot", "orc_read_slot"):
            getattr(lib, name).restype = C.c_size_t
        lib.orc_capacity_tokens.argtypes = [C.c_uint32, C.c_int]
        lib.orc_write_slot.argtypes = [C.c_uint32, C.c_int, C.c_uint]
        lib.orc_read_slot.argtypes = [C.c_uint32, C.c_int, C.c_uint]
        lib.orc_synth_samples.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        lib.orc_random_taps.argtypes = [C.c_uint64, C.c_uint, C.c_void_p]
        lib.orc_random_schedule.argtypes = [C.c_size_t, C.c_uint64, C.c_void_p]
        lib.orc_synth_bytes.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        lib.orc_motion_gray.argtypes = [C.c_void_p, C.c_size_t, C.c_uint, C.c_uint, C.c_uint8, C.c_void_p]
        lib.orc_motion_rgb.argtypes = [C.c_void_p, C.c_size_t, C.c_uint, C.c_uint, C.c_uint8, C.c_void_p,
                                       C.c_void_p]
        lib.orc_rgb_to_gray.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        lib.orc_gauss5x5.argtypes = [C.c_void_p, C.c_void_p, C.c_uint, C.c_uint]
        lib.orc_median5.argtypes = [C.c_void_p, C.c_void_p, C.c_uint, C.c_uint]
        lib.orc_thres_diff.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_uint, C.c_uint8]
        lib.orc_poly_branch.argtypes = [C.c_uint, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        lib.orc_fir.argtypes = [C.c_uint, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_size_t, C.c_void_p, C.c_void_p]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_PATH} missing (reference not built: needs /root/reference at build time)")
        lib = C.CDLL(REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_hardware_concurrency.restype = C.c_uint
        lib.ref_synth_samples.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        lib.ref_random_taps.argtypes = [C.c_uint64, C.c_void_p]
        lib.ref_random_schedule.argtypes = [C.c_size_t, C.c_uint64, C.c_void_p]
        lib.ref_synth_frames.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.c_uint64, C.c_void_p]
        lib.ref_check_config.argtypes = [C.c_uint16]
        lib.ref_poly_branch.argtypes = [C.c_uint, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
        lib.ref_fir10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                  C.c_void_p]
        lib.ref_oracle_dpd.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32,
                                       C.c_void_p]
        lib.ref_dpd_network.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32,
                                        C.c_void_p, _dp, _dp]
        lib.ref_gauss5x5.argtypes = [C.c_void_p, C.c_void_p, C.c_uint, C.c_uint]
        lib.ref_median5.argtypes = [C.c_void_p, C.c_void_p, C.c_uint, C.c_uint]
        lib.ref_thres_diff.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_uint, C.c_uint8]
        lib.ref_oracle_motion.argtypes = [C.c_void_p, C.c_size_t, C.c_uint, C.c_uint, C.c_uint8, C.c_void_p]
        lib.ref_motion_network.argtypes = [C.c_void_p, C.c_size_t, C.c_uint, C.c_uint, C.c_uint8, C.c_uint32,
                                           C.c_void_p, _dp, _dp]
        for name in ("ref_capacity_tokens", "ref_write_slot", "ref_read_slot"):
            getattr(lib, name).restype = C.c_size_t
        lib.ref_capacity_tokens.argtypes = [C.c_uint32, C.c_int]
        lib.ref_write_slot.argtypes = [C.c_uint32, C.c_int, C.c_uint]
        lib.ref_read_slot.argtypes = [C.c_uint32, C.c_int, C.c_uint]
        lib.ref_parse_schedule.restype = C.c_long
        lib.ref_parse_schedule.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t]
        lib.ref_parse_taps.argtypes = [C.c_char_p, C.c_void_p]
        lib.ref_mem_total.restype = C.c_uint64
        lib.ref_mem_total.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_uint32, C.c_uint32]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- generators
def synth_samples(n: int, seed: int) -> np.ndarray:
    """Interleaved complex64 samples, proj/src/dpd.cpp:496-505."""
    out = np.empty(2 * n, np.float32)
    port().orc_synth_samples(n, seed, _ptr(out))
    return out


def random_taps(seed: int, T: int = 10) -> np.ndarray:
    """(10, T, 2) float32 taps, proj/src/dpd.cpp:485-494 (T-generic stream)."""
    out = np.empty(10 * T * 2, np.float32)
    port().orc_random_taps(seed, T, _ptr(out))
    return out.reshape(10, T, 2)


def random_schedule(entries: int, seed: int) -> np.ndarray:
    out = np.empty(entries, np.uint16)
    port().orc_random_schedule(entries, seed, _ptr(out))
    return out


def synth_bytes(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    port().orc_synth_bytes(n, seed, _ptr(out))
    return out


def first_n(k: int) -> int:
    return (1 << k) - 1


# ---------------------------------------------------------------- DPD
def dpd(inp: np.ndarray, taps: np.ndarray, schedule, period: int) -> np.ndarray:
    """oracle_dpd restated (proj/src/dpd.cpp:358-391), T from taps.shape[1]."""
    inp = np.ascontiguousarray(inp, np.float32).reshape(-1)
    taps = np.ascontiguousarray(taps, np.float32)
    T = taps.shape[1]
    sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    n = inp.size // 2
    out = np.empty_like(inp)
    rc = port().orc_dpd(_ptr(inp), n, _ptr(taps), T, _ptr(sched), sched.size, period, _ptr(out))
    if rc != 0:
        raise ValueError("oracle_dpd: bad schedule or period")
    return out


def _threads(threads):
    return threads or max(1, len(os.sched_getaffinity(0)))


def dpd_mt(inp: np.ndarray, taps: np.ndarray, schedule, period: int, threads: int | None = None) -> np.ndarray:
    """oracle_dpd over block ranges in parallel; bit-identical to dpd()."""
    inp = np.ascontiguousarray(inp, np.float32).reshape(-1)
    taps = np.ascontiguousarray(taps, np.float32)
    sched = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    out = np.empty_like(inp)
    rc = port().orc_dpd_mt(_ptr(inp), inp.size // 2, _ptr(taps), taps.shape[1], _ptr(sched), sched.size, period,
                           _ptr(out), _threads(threads))
    if rc != 0:
        raise ValueError("oracle_dpd: bad schedule or period")
    return out


def motion_mt(frames: np.ndarray, w: int, h: int, fmt: int = 3, threshold: int = 32, prev_rgb=None,
              threads: int | None = None) -> np.ndarray:
    """motion_rgb (fmt 3) / motion_gray (fmt 1) over frame ranges in parallel; bit-identical."""
    frames = np.ascontiguousarray(frames, np.uint8).reshape(-1)
    count = frames.size // (fmt * w * h)
    out = np.empty(count * w * h, np.uint8)
    prev = None if prev_rgb is None else np.ascontiguousarray(prev_rgb, np.uint8).reshape(-1)
    port().orc_motion_mt(_ptr(frames), count, w, h, fmt, threshold, None if prev is None else _ptr(prev), _ptr(out),
                         _threads(threads))
    return out


def compare_samples(got: np.ndarray, want: np.ndarray, tol: float = 1e-5):
    """proj/src/bench.cpp:307-326; returns (first_bad_index or -1, worst_rel_err)."""
    got = np.ascontiguousarray(got, np.float32).reshape(-1)
    want = np.ascontiguousarray(want, np.float32).reshape(-1)
    assert got.size == want.size
    worst = C.c_double(0)
    idx = port().orc_compare_samples(_ptr(got), _ptr(want), got.size // 2, tol, C.byref(worst))
    return int(idx), float(worst.value)


# ---------------------------------------------------------------- motion
def motion_gray(frames: np.ndarray, w: int, h: int, threshold: int = 32) -> np.ndarray:
    frames = np.ascontiguousarray(frames, np.uint8).reshape(-1)
    out = np.empty_like(frames)
    port().orc_motion_gray(_ptr(frames), frames.size // (w * h), w, h, threshold, _ptr(out))
    return out


def motion_rgb(rgb: np.ndarray, w: int, h: int, threshold: int = 32, prev_rgb=None) -> np.ndarray:
    rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
    count = rgb.size // (3 * w * h)
    out = np.empty(count * w * h, np.uint8)
    prev = None if prev_rgb is None else np.ascontiguousarray(prev_rgb, np.uint8).reshape(-1)
    port().orc_motion_rgb(_ptr(rgb), count, w, h, threshold, None if prev is None else _ptr(prev), _ptr(out))
    return out


def rgb_to_gray(rgb: np.ndarray) -> np.ndarray:
    rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
    out = np.empty(rgb.size // 3, np.uint8)
    port().orc_rgb_to_gray(_ptr(rgb), out.size, _ptr(out))
    return out


def gauss5x5(img: np.ndarray, w: int, h: int) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8).reshape(-1)
    out = np.empty_like(img)
    port().orc_gauss5x5(_ptr(img), _ptr(out), w, h)
    return out


def median5(img: np.ndarray, w: int, h: int) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8).reshape(-1)
    out = np.empty_like(img)
    port().orc_median5(_ptr(img), _ptr(out), w, h)
    return out


def thres_diff(prev: np.ndarray, cur: np.ndarray, w: int, h: int, threshold: int) -> np.ndarray:
    prev = np.ascontiguousarray(prev, np.uint8).reshape(-1)
    cur = np.ascontiguousarray(cur, np.uint8).reshape(-1)
    out = np.empty_like(cur)
    port().orc_thres_diff(_ptr(prev), _ptr(cur), _ptr(out), w, h, threshold)
    return out


# ---------------------------------------------------------------- channel
def capacity_tokens(rate: int, has_delay: bool) -> int:
    return int(port().orc_capacity_tokens(rate, int(has_delay)))


def write_slot(rate: int, has_delay: bool, phase: int) -> int:
    return int(port().orc_write_slot(rate, int(has_delay), phase))


def read_slot(rate: int, has_delay: bool, phase: int) -> int:
    return int(port().orc_read_slot(rate, int(has_delay), phase))
