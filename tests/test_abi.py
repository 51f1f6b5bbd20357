"""CPU: the C-ABI library loads, exports every symbol include/df_cuda.h
declares, and its host-side logic (slot arithmetic, argument validation)
behaves like the reference -- no compute calls (no GPU here)."""
import ctypes as C

import pytest

import paper_1611_03226_b200 as P
from oracle import oracle as O


def test_library_exports_every_header_symbol():
    lib = P.lib()
    syms = P.header_symbols()
    assert len(syms) > 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_signatures_cover_header():
    from paper_1611_03226_b200 import _lib
    assert set(_lib._SIGS) == set(P.header_symbols())


def test_abi_version():
    assert P.lib().df_abi_version() == 1


@pytest.mark.parametrize("rate", [1, 2, 3, 4, 7, 16])
@pytest.mark.parametrize("delay", [False, True])
def test_slot_arithmetic_matches_reference(rate, delay):
    lib = P.lib()
    assert lib.df_slot_capacity(rate, int(delay)) == O.capacity_tokens(rate, delay)
    for phase in range(7):
        assert lib.df_slot_write_first(rate, int(delay), phase) == O.write_slot(rate, delay, phase)
        assert lib.df_slot_read_first(rate, int(delay), phase) == O.read_slot(rate, delay, phase)


def test_argument_validation_maps_to_reference_exceptions():
    from paper_1611_03226_b200 import _lib
    lib = P.lib()
    h = C.c_void_p()
    # proj/src/channel.cpp:38-40 invalid_argument for rate 0
    rc = lib.df_channel_create(0, 8, 0, 0, None, C.byref(h))
    assert rc == _lib.DF_EINVAL and b"token_rate" in lib.df_last_error()
    rc = lib.df_channel_create(0, 8, 1, 0, b"x" * 8, C.byref(h))
    assert rc == _lib.DF_EINVAL
    taps = (C.c_float * 200)()
    assert lib.df_dpd_create(0, 0, 10, taps, C.byref(h)) == _lib.DF_EINVAL      # period 0
    assert lib.df_dpd_create(0, 64, 33, taps, C.byref(h)) == _lib.DF_EINVAL     # T > 32
    assert lib.df_motion_create(0, 4, 10, 1, 32, C.byref(h)) == _lib.DF_EINVAL  # below 5x5
    assert lib.df_motion_create(0, 10, 10, 2, 32, C.byref(h)) == _lib.DF_EINVAL  # bad format
    with pytest.raises(P.InvalidArgument):
        _lib.check(_lib.DF_EINVAL)


def test_no_cpu_fallback_without_device():
    if P.device_count() > 0:
        pytest.skip("a device is visible")
    from paper_1611_03226_b200 import dpd
    with pytest.raises(P.CudaError):
        dpd.DpdActor(64, O.random_taps(1))


def test_shard_entry_points_validate_arguments():
    """df_*_fire_halo, df_ipc_* and df_halo_copy reject null handles/buffers
    with DF_EINVAL before touching a device."""
    from paper_1611_03226_b200 import _lib
    lib = P.lib()
    tails = (C.c_void_p * 10)()
    buf = C.c_void_p(0x1000)
    assert lib.df_motion_fire_halo(None, buf, buf, buf, 4, None) == _lib.DF_EINVAL
    assert lib.df_dpd_fire_halo(None, tails, buf, buf, buf, 4, None) == _lib.DF_EINVAL
    assert lib.df_ipc_get_handle(None, None) == _lib.DF_EINVAL
    assert lib.df_ipc_open_handle(0, None, None) == _lib.DF_EINVAL
    assert lib.df_ipc_handle_size() == 64  # cudaIpcMemHandle_t
    assert b"null" in lib.df_last_error()
