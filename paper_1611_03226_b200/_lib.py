"""ctypes binding of libdf_cuda.so (the C ABI declared in include/df_cuda.h).

This module only marshals arguments; every computation happens in the
CUDA library.  There is no CPU fallback: if the library is missing, or a
compute call is made without a CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DF_CUDA_LIB", os.path.join(HERE, "libdf_cuda.so"))
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "df_cuda.h")

DF_OK, DF_EINVAL, DF_ELOGIC, DF_EABORTED, DF_ECUDA, DF_ECONTROL, DF_EOS, DF_ETIMEOUT = range(8)
DF_MOTION_GRAY, DF_MOTION_RGB = 1, 3


class DfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(DfError, ValueError):
    """DF_EINVAL -- std::invalid_argument in the reference."""


class LogicError(DfError):
    """DF_ELOGIC -- std::logic_error (contract misuse) in the reference."""


class RunAborted(DfError):
    """DF_EABORTED -- dynflow::RunAborted."""


class ControlError(DfError):
    """DF_ECONTROL -- dynflow::ControlError / check_config rejection."""


class CudaError(DfError):
    pass


class EndOfStream(DfError):
    """DF_EOS -- read_start on a closed, drained channel (nullopt)."""


class WatchdogTimeout(DfError):
    """DF_ETIMEOUT -- a device-resident actor waited past the run's timeout."""


_EXC = {DF_EINVAL: InvalidArgument, DF_ELOGIC: LogicError, DF_EABORTED: RunAborted,
        DF_ECUDA: CudaError, DF_ECONTROL: ControlError, DF_EOS: EndOfStream, DF_ETIMEOUT: WatchdogTimeout}


class DfChanStats(C.Structure):
    _fields_ = [("tokens_written", C.c_uint64), ("tokens_read", C.c_uint64),
                ("tokens_available", C.c_uint64), ("write_phase", C.c_uint32),
                ("read_phase", C.c_uint32), ("closed", C.c_uint32), ("error", C.c_uint32)]


class DfRegion(C.Structure):
    _fields_ = [("dptr", C.c_void_p), ("first_slot", C.c_size_t), ("tokens", C.c_size_t),
                ("serial", C.c_uint64), ("direction", C.c_int)]


_vp, _sz, _u32, _u64, _i, _u8, _u16 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_int, C.c_uint8, C.c_uint16
_P = C.POINTER

# name -> (restype, argtypes)
_SIGS = {
    "df_last_error": (C.c_char_p, []),
    "df_abi_version": (_i, []),
    "df_device_count": (_i, [_P(_i)]),
    "df_device_sm_count": (_i, [_i, _P(_i)]),
    "df_set_device": (_i, [_i]),
    "df_stream_create": (_i, [_i, _P(_vp)]),
    "df_stream_destroy": (_i, [_vp]),
    "df_stream_synchronize": (_i, [_vp]),
    "df_event_create": (_i, [_P(_vp)]),
    "df_event_destroy": (_i, [_vp]),
    "df_event_record": (_i, [_vp, _vp]),
    "df_event_synchronize": (_i, [_vp]),
    "df_event_elapsed_ms": (_i, [_vp, _vp, _P(C.c_float)]),
    "df_stream_wait_event": (_i, [_vp, _vp]),
    "df_malloc": (_i, [_i, _sz, _P(_vp)]),
    "df_free": (_i, [_vp]),
    "df_host_alloc": (_i, [_sz, _P(_vp)]),
    "df_host_free": (_i, [_vp]),
    "df_memcpy_h2d": (_i, [_vp, _vp, _sz, _vp]),
    "df_memcpy_d2h": (_i, [_vp, _vp, _sz, _vp]),
    "df_memcpy_d2d": (_i, [_vp, _vp, _sz, _vp]),
    "df_memset": (_i, [_vp, _i, _sz, _vp]),
    "df_channel_create": (_i, [_i, _sz, _u32, _i, _vp, _P(_vp)]),
    "df_channel_destroy": (_i, [_vp]),
    "df_channel_capacity_tokens": (_sz, [_vp]),
    "df_channel_capacity_bytes": (_sz, [_vp]),
    "df_channel_token_size": (_sz, [_vp]),
    "df_channel_token_rate": (_u32, [_vp]),
    "df_channel_has_delay": (_i, [_vp]),
    "df_channel_storage": (_vp, [_vp]),
    "df_channel_device_state": (_vp, [_vp]),
    "df_slot_capacity": (_sz, [_u32, _i]),
    "df_slot_write_first": (_sz, [_u32, _i, C.c_uint]),
    "df_slot_read_first": (_sz, [_u32, _i, C.c_uint]),
    "df_channel_write_start": (_i, [_vp, _sz, _P(DfRegion)]),
    "df_channel_write_end": (_i, [_vp, _P(DfRegion), _vp]),
    "df_channel_read_start": (_i, [_vp, _sz, _P(DfRegion)]),
    "df_channel_read_end": (_i, [_vp, _P(DfRegion), _vp]),
    "df_channel_close": (_i, [_vp, _vp]),
    "df_channel_abort": (_i, [_vp]),
    "df_channel_stats": (_i, [_vp, _P(DfChanStats)]),
    "df_channel_check": (_i, [_vp]),
    "df_channel_test_produce": (_i, [_vp, _u64, _u32, _u64, _vp]),
    "df_channel_test_consume": (_i, [_vp, _u64, _u32, _u64, _i, _vp, _vp]),
    "df_dpd_create": (_i, [_i, _u32, _u32, _vp, _P(_vp)]),
    "df_dpd_destroy": (_i, [_vp]),
    "df_dpd_set_taps": (_i, [_vp, _vp, _vp]),
    "df_dpd_reset": (_i, [_vp, _vp]),
    "df_dpd_kernel_name": (C.c_char_p, [_vp]),
    "df_dpd_get_state": (_i, [_vp, _vp]),
    "df_dpd_error": (_i, [_vp]),
    "df_dpd_set_history": (_i, [_vp, _vp, _u32, _u32, _vp]),
    "df_dpd_fire": (_i, [_vp, _vp, _vp, _vp, _u64, _vp]),
    "df_dpd_fire_halo": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _vp]),
    "df_dpd_fire_channels": (_i, [_vp, _vp, _vp, _vp, _u32, _vp]),
    "df_dpd_config_tokens": (_i, [_i, _vp, _sz, _u64, _u64, _vp, _vp]),
    "df_dpd_run_host": (_i, [_vp, _vp, _vp, _u64, _vp, _sz, _u64, _vp]),
    "df_motion_create": (_i, [_i, C.c_uint, C.c_uint, _i, _u8, _P(_vp)]),
    "df_motion_destroy": (_i, [_vp]),
    "df_motion_set_prev_frame": (_i, [_vp, _vp, _vp]),
    "df_motion_fire": (_i, [_vp, _vp, _vp, _u32, _vp]),
    "df_motion_fire_halo": (_i, [_vp, _vp, _vp, _vp, _u32, _vp]),
    "df_motion_fire_channels": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "df_motion_run_host": (_i, [_vp, _vp, _vp, _u64, _u32, _vp]),
    "df_motion_gauss5x5": (_i, [_vp, _vp, C.c_uint, C.c_uint, _vp]),
    "df_motion_thres_diff": (_i, [_vp, _vp, _vp, C.c_uint, C.c_uint, _u8, _vp]),
    "df_motion_median5": (_i, [_vp, _vp, C.c_uint, C.c_uint, _vp]),
    "df_motion_rgb_to_gray": (_i, [_vp, _vp, _sz, _vp]),
    "df_motion_kernel_name": (C.c_char_p, [_vp]),
    "df_launch_host_func": (_i, [_vp, _vp, _vp]),
    "df_peer_enable": (_i, [_i, _i]),
    "df_halo_copy": (_i, [_i, _vp, _i, _vp, _sz, _vp]),
    "df_ipc_handle_size": (_i, []),
    "df_ipc_get_handle": (_i, [_vp, _vp]),
    "df_ipc_open_handle": (_i, [_i, _vp, _P(_vp)]),
    "df_ipc_close_handle": (_i, [_vp]),
    "df_net_create": (_i, [_i, _P(_vp)]),
    "df_net_destroy": (_i, [_vp]),
    "df_net_add_actor": (_i, [_vp, _i, _vp, _sz, _u32, _vp, _vp, _sz, _vp, _sz, _u64, _P(_i)]),
    "df_net_set_control_table": (_i, [_vp, _i, _vp, _u32]),
    "df_net_run": (_i, [_vp, C.c_double]),
    "df_net_abort": (_i, [_vp]),
    "df_net_fault": (_i, [_vp, _P(_i), _P(_i), _P(_u32)]),
    "df_net_actor_stats": (_i, [_vp, _i, _P(_u64), _P(C.c_double)]),
    "df_net_actor_profile": (_i, [_vp, _i, _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "df_fill_random_u8": (_i, [_vp, _sz, _u64, _vp]),
    "df_fill_random_pm1": (_i, [_vp, _sz, _u64, _vp]),
    "df_kernel_launches": (_u64, []),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function declared in include/df_cuda.h."""
    text = open(HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(df_[a-z0-9_]+)\s*\(", text)))


def lib():
    """Loads libdf_cuda.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(make -C paper_1611_03226_b200/csrc). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != DF_OK:
        msg = lib().df_last_error().decode(errors="replace")
        raise _EXC.get(rc, DfError)(rc, msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().df_device_count(C.byref(n))
    return n.value if rc == DF_OK else 0


def require_gpu():
    if device_count() < 1:
        raise CudaError(DF_ECUDA, "no CUDA device visible: the GPU-actor path has no CPU fallback")
