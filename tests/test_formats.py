"""CPU: the data formats either side of the GPU-actor path (
include/df/io.hpp, df::dpd::parse_schedule / parse_taps) through the C ABI
of libdf_host.so.  Parsers are checked against the reference's own
(proj/src/dpd.cpp:393-462, via oracle/_ref) on valid and invalid inputs;
the file formats follow proj/src/bench.cpp:25-97 and :173-262."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1611_03226_b200 import host_api as H

ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")

SCHEDULES = [
    "2\n",
    "10\n",
    "3: 1,5,9\n# comment line\n\n2:10,1  # trailing comment\n4\n",
    "  7  \n5 : 2 , 4 , 6 , 8 , 10\n",
]
BAD_SCHEDULES = [
    "",                      # no entries
    "# only a comment\n",
    "1\n",                   # k < 2
    "11\n",
    "3: 1,2\n",              # too few indices
    "2: 1;2\n",              # bad separator
    "2: 1,11\n",             # branch out of range
    "2: 3,3\n",              # listed twice
    "2 x\n",                 # expected ':'
]


def _ref_schedule(text):
    R = O.ref()
    out = np.zeros(64, np.uint16)
    n = R.ref_parse_schedule(text.encode(), out.ctypes.data, out.size)
    return None if n < 0 else out[:n], R.ref_last_error().decode()


@ref_only
@pytest.mark.parametrize("text", SCHEDULES)
def test_parse_schedule_equals_reference(text):
    want, _ = _ref_schedule(text)
    assert want is not None
    np.testing.assert_array_equal(H.parse_schedule(text), want)


@ref_only
@pytest.mark.parametrize("text", BAD_SCHEDULES)
def test_parse_schedule_rejects_what_the_reference_rejects(text):
    want, ref_msg = _ref_schedule(text)
    assert want is None
    with pytest.raises(H.HostRunError) as e:
        H.parse_schedule(text)
    assert ref_msg in str(e.value)  # the reference's message, verbatim


def test_parse_schedule_values():
    np.testing.assert_array_equal(H.parse_schedule("2\n3: 1,5,9\n10\n"),
                                  np.array([0b11, 0b100010001, 0x3FF], np.uint16))


def _taps_text(taps, T=10):
    return "\n".join(" ".join(f"{float(taps[b, k, 0]):.9g},{float(taps[b, k, 1]):.9g}" for k in range(T))
                     for b in range(10)) + "\n"


@ref_only
def test_parse_taps_equals_reference():
    rng = np.random.default_rng(5)
    taps = rng.uniform(-1, 1, (10, 10, 2)).astype(np.float32)
    text = "# taps\n\n" + _taps_text(taps).replace("\n", "  # b\n", 3)
    out = np.zeros((10, 10, 2), np.float32)
    assert O.ref().ref_parse_taps(text.encode(), out.ctypes.data) == 0
    got = H.parse_taps(text)
    assert np.array_equal(got.view(np.uint32), out.view(np.uint32))
    assert np.array_equal(got, taps)


@ref_only
@pytest.mark.parametrize("text", [
    "1,0 " * 10 + "\n",                            # 1 branch only
    ("1,0 " * 9 + "\n") + ("1,0 " * 10 + "\n") * 9,  # 9 taps in branch 1
    ("1,0 " * 11 + "\n") * 10,                     # 11 taps
    ("1;0 " * 10 + "\n") * 10,                     # malformed pair
])
def test_parse_taps_rejects_what_the_reference_rejects(text):
    out = np.zeros(200, np.float32)
    assert O.ref().ref_parse_taps(text.encode(), out.ctypes.data) != 0
    ref_msg = O.ref().ref_last_error().decode()
    with pytest.raises(H.HostRunError) as e:
        H.parse_taps(text)
    assert ref_msg in str(e.value)


def test_parse_taps_32_extension():
    taps = np.random.default_rng(6).uniform(-0.5, 0.5, (10, 32, 2)).astype(np.float32)
    got = H.parse_taps(_taps_text(taps, 32), 32)
    assert np.array_equal(got, taps)
    with pytest.raises(H.HostRunError):
        H.parse_taps(_taps_text(taps, 32), 10)  # more than 10 entries


def test_pgm_round_trip_and_multi_frame(tmp_path):
    f = O.synth_bytes(3 * 37 * 11, 9).reshape(3, 11, 37)
    p = str(tmp_path / "a.pgm")
    H.write_pgm(p, f, 37, 11)
    px, w, h = H.read_pgm(p)
    assert (w, h) == (37, 11)
    assert np.array_equal(px, f)
    # Header comments and odd whitespace, as netpbm allows (bench.cpp:54-71).
    q = tmp_path / "b.pgm"
    q.write_bytes(b"P5 # made by hand\n37\t11\n# maxval next\n255\n" + f[0].tobytes() + b"\n\n" +
                  b"P5\n37 11\n255\n" + f[1].tobytes())
    px, w, h = H.read_pgm(str(q))
    assert px.shape == (2, 11, 37) and np.array_equal(px, f[:2])


@pytest.mark.parametrize("data,what", [
    (b"P2\n2 2\n255\n0 0 0 0", "not binary PGM"),
    (b"P5\n2 2\n65535\n" + bytes(8), "maxval must be 255"),
    (b"P5\n2 2\n255\n" + bytes(3), "truncated PGM data"),
    (b"P5\n2 2", "truncated PGM header"),
    (b"P5\n2 2\n255\n" + bytes(4) + b"P5\n3 2\n255\n" + bytes(6), "change dimensions"),
    (b"", "holds no PGM frames"),
])
def test_pgm_errors(tmp_path, data, what):
    p = tmp_path / "bad.pgm"
    p.write_bytes(data)
    with pytest.raises(H.HostRunError) as e:
        H.read_pgm(str(p))
    assert what in str(e.value) and "[8]" in str(e.value)  # FormatError (the reference's ConfigError)


def test_missing_file_is_format_error(tmp_path):
    with pytest.raises(H.HostRunError) as e:
        H.read_cf32(str(tmp_path / "nope.cf32"))
    assert "cannot open" in str(e.value) and "[8]" in str(e.value)


def test_raw_frames_and_cf32(tmp_path):
    rgb = O.synth_bytes(4 * 16 * 8 * 3, 3)
    p = str(tmp_path / "f.rgb")
    H.write_file(p, rgb)
    assert np.array_equal(H.read_raw_frames(p, 16, 8, 3), rgb)
    with pytest.raises(H.HostRunError) as e:
        H.read_raw_frames(p, 16, 9, 3)
    assert "multiple of 432-byte frames" in str(e.value)
    x = O.synth_samples(1000, 4)
    q = str(tmp_path / "x.cf32")
    H.write_file(q, x)
    assert np.array_equal(H.read_cf32(q).view(np.uint32), x.view(np.uint32))
    (tmp_path / "odd.cf32").write_bytes(bytes(12))
    with pytest.raises(H.HostRunError) as e:
        H.read_cf32(str(tmp_path / "odd.cf32"))
    assert "interleaved float re,im pairs" in str(e.value)


def test_config_token_wire_form():
    # dpd.cpp:38-47: 4 bytes little endian; decode keeps the low 16 bits
    for m in (0x3, 0x3FF, 0x155, 0x8001):
        assert H.encode_config(m) == m.to_bytes(4, "little")
        assert H.decode_config(m.to_bytes(4, "little")) == m
    assert H.decode_config((0x12345).to_bytes(4, "little")) == 0x2345


def test_library_generators_match_the_reference_streams(hashes):
    # df::dpd::random_schedule / random_taps / synth_samples and
    # df::motion::synth_frames against the reference's own streams (golden
    # values recorded from the compiled reference, tests/golden).
    import hashlib
    g = hashes["generators"]
    assert H.synth("taps", 10, 808).tolist() == g["taps808"]
    assert H.synth("schedule", 16, 809).tolist() == g["sched16_809"]
    assert H.synth("frames", 320 * 240, 606)[:64].tolist() == g["frames_606_first64"]
    x = H.synth("samples", 1 << 20, 810)
    assert hashlib.sha256(x.tobytes()).hexdigest() == hashes["dpd_acceptance8"]["input_sha256"]
