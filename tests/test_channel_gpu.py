"""GPU: device-resident channels keep the reference Channel's semantics --
Eq. 1 capacity, Fig. 2 slot walk with the phase-2 copy-back, FIFO stream
equivalence, and its contract errors (proj/tests/test_channel.cpp,
proj/tests/acceptance.cpp [1]-[3])."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def splitmix64(x):
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def fill_token(size, seed, index):
    # proj/tests/acceptance.cpp:62-66
    return np.array([splitmix64(seed ^ ((index * 1315423911 + i) & ((1 << 64) - 1))) & 0xFF
                     for i in range(size)], np.uint8)


def h2d(dptr, arr, s):
    from paper_1611_03226_b200._lib import call
    call("df_memcpy_h2d", C.c_void_p(dptr), arr.ctypes.data_as(C.c_void_p), arr.nbytes, s.handle)


def d2h(arr, dptr, s):
    from paper_1611_03226_b200._lib import call
    call("df_memcpy_d2h", arr.ctypes.data_as(C.c_void_p), C.c_void_p(dptr), arr.nbytes, s.handle)


@pytest.mark.parametrize("r", [1, 2, 3, 4, 8, 16])
def test_capacity_rule(gpu, r):
    from paper_1611_03226_b200.channel import DeviceChannel
    for s in (1, 76800):
        d = DeviceChannel(s, r, True)
        g = DeviceChannel(s, r, False)
        assert d.capacity_tokens == O.capacity_tokens(r, True) == 3 * r + 1
        assert g.capacity_tokens == 2 * r
        assert d.capacity_bytes == (3 * r + 1) * s and g.capacity_bytes == 2 * r * s


def test_delay_pattern_replay_acceptance2(gpu):
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Stream
    s = Stream()
    tok = 8
    ch = DeviceChannel(tok, 4, True)
    value = 1
    for phase, (ws, rs) in enumerate([(1, 0), (5, 4), (9, 8)]):
        w = ch.write_start(4)
        assert w.first_slot == ws and w.tokens == 4
        data = np.concatenate([fill_token(tok, 9, value + t) for t in range(4)])
        value += 4
        h2d(w.dptr, data, s)
        ch.write_end(w, s)
        rd = ch.read_start(4)
        assert rd.first_slot == rs
        ch.read_end(rd, s)
    w = ch.write_start(4)
    assert w.first_slot == 1
    h2d(w.dptr, np.concatenate([fill_token(tok, 9, value + t) for t in range(4)]), s)
    ch.write_end(w, s)
    rd = ch.read_start(4)
    assert rd.first_slot == 0
    first = np.empty(tok, np.uint8)
    d2h(first, rd.dptr, s)
    s.synchronize()
    np.testing.assert_array_equal(first, fill_token(tok, 9, 12))  # slot 12 -> slot 0 copy
    ch.read_end(rd, s)
    ch.check()


@pytest.mark.parametrize("rate", [1, 4, 7])
@pytest.mark.parametrize("delay", [False, True])
def test_device_stream_equivalence(gpu, rate, delay):
    """Producer and consumer GPU actors on separate streams resolve their
    regions from the device phases; the consumer checks every byte against
    the reference's token generator (criterion [3] pattern)."""
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Buffer, Event, Stream
    tok, firings, seed = 16, 3000 // rate, 77 + rate + (1000 if delay else 0)
    ch = DeviceChannel(tok, rate, delay)
    sp, sc = Stream(), Stream()
    bad = Buffer(8)
    bad.zero()
    # Stream-ordered schedule: producer firing i after consumer firing i-2
    # (capacity 2 phases) and consumer firing i after producer firing i.
    ev_p = [Event() for _ in range(firings)]
    ev_c = [Event() for _ in range(firings)]
    from paper_1611_03226_b200._lib import call
    produced = 0
    consumed_pos = 0
    for i in range(firings):
        if i >= 2:
            call("df_stream_wait_event", sp.handle, ev_c[i - 2].handle)
        ch.test_produce(produced, 1, seed, sp)
        produced += rate
        ev_p[i].record(sp)
        call("df_stream_wait_event", sc.handle, ev_p[i].handle)
        ch.test_consume(consumed_pos, 1, seed, delay, bad.ptr, sc)
        consumed_pos += rate
        ev_c[i].record(sc)
    sc.synchronize()
    sp.synchronize()
    assert int(bad.download(np.uint64)[0]) == 0
    st = ch.stats()
    assert st.error == 0
    assert st.tokens_written == firings * rate and st.tokens_read == firings * rate
    assert st.tokens_available == (1 if delay else 0)


def test_contract_errors(gpu):
    from paper_1611_03226_b200 import LogicError
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Stream
    s = Stream()
    ch = DeviceChannel(4, 2)
    with pytest.raises(LogicError):
        ch.write_start(1)  # n != r (proj/src/channel.cpp:65-68)
    w = ch.write_start(2)
    with pytest.raises(LogicError):
        ch.write_start(2)  # outstanding write
    ch.write_end(w, s)
    with pytest.raises(LogicError):
        ch.write_end(w, s)  # no matching start
    ch.close_stream(s)
    with pytest.raises(LogicError):
        ch.write_start(2)  # write after close
    s.synchronize()
    assert ch.stats().closed == 1


def test_device_detects_overflow(gpu):
    """A schedule that writes a third phase into a 2r buffer before any read
    is caught on the device (the reference would block)."""
    from paper_1611_03226_b200 import LogicError
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Stream
    s = Stream()
    ch = DeviceChannel(4, 1)
    ch.test_produce(0, 3, 1, s)
    s.synchronize()
    with pytest.raises(LogicError):
        ch.check()


@pytest.mark.parametrize("rate", [1, 4])
@pytest.mark.parametrize("delay", [False, True])
def test_channel_class_api(gpu, rate, delay):
    # df::Channel (include/df/channel.hpp): the reference's Channel calls over
    # a device channel -- FIFO order (a delay channel first yields its initial
    # token), n != rate -> logic_error, counters, end of stream after close,
    # RunAborted after abort (proj/include/dynflow/channel.hpp:71-135).
    from paper_1611_03226_b200 import host_api as H
    firings = 5
    out, status = H.channel_class_demo(rate, delay, firings)
    stream = np.arange(1, firings * rate + 1, dtype=np.uint32)
    if delay:  # the delay token shifts the stream by one token (Fig. 2)
        stream = np.concatenate([[0xFFFFFFFF], stream[:-1]]).astype(np.uint32)
    np.testing.assert_array_equal(out, stream)
    assert status == 1 | 2 | 4 | 8, status
