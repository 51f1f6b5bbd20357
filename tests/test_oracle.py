"""CPU: the oracle restatement (oracle/oracle.c) against the reference's own
outputs -- committed golden fixtures always, and the reference compiled
from /root/reference (oracle/_ref) when it was built."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_generators_match_reference_streams(hashes):
    g = hashes["generators"]
    assert O.random_taps(808).reshape(-1).tolist() == g["taps808"]
    assert O.random_schedule(16, 809).tolist() == g["sched16_809"]
    assert O.synth_bytes(320 * 240, 606)[:64].tolist() == g["frames_606_first64"]
    assert sha(O.synth_samples(1 << 20, 810)) == hashes["dpd_acceptance8"]["input_sha256"]


@pytest.mark.parametrize("name", ["net_p256_s41", "gating_p64", "short_p4", "counts_p16"])
def test_dpd_oracle_equals_reference_fixture(small, name):
    x, taps, sched = small[f"dpd_{name}_in"], small[f"dpd_{name}_taps"], small[f"dpd_{name}_sched"]
    period = int(small[f"dpd_{name}_period"][0])
    got = O.dpd(x, taps, sched, period)
    np.testing.assert_array_equal(bits(got), bits(small[f"dpd_{name}_out"]))


@pytest.mark.parametrize("k", [1, 2, 10])
def test_dpd_oracle_single_and_full_masks(small, k):
    got = O.dpd(small["dpd_k_in"], small["dpd_k_taps"], [(1 << k) - 1], 64)
    np.testing.assert_array_equal(bits(got), bits(small[f"dpd_k{k}_out"]))


def test_dpd_acceptance8_hash(hashes):
    h = hashes["dpd_acceptance8"]
    x = O.synth_samples(h["samples"], h["input_seed"])
    y = O.dpd(x, O.random_taps(h["taps_seed"]), O.random_schedule(*h["sched"]), h["period"])
    assert sha(y) == h["out_sha256"]


def test_dpd_p4096_random_hash(hashes):
    h = hashes["dpd_p4096_random"]
    x = O.synth_samples(h["samples"], h["input_seed"])
    y = O.dpd(x, O.random_taps(h["taps_seed"]), O.random_schedule(*h["sched"]), h["period"])
    assert sha(y) == h["out_sha256"]


def test_motion_oracle_fixtures(small):
    got = O.motion_gray(small["motion_64x48_in"], 64, 48)
    np.testing.assert_array_equal(got, small["motion_64x48_out"])
    for thr in (0, 32, 127, 128, 254):
        got = O.motion_gray(small["motion_33x29_in"], 33, 29, thr)
        np.testing.assert_array_equal(got, small[f"motion_33x29_t{thr}_out"])


def test_motion_acceptance6_hash(hashes):
    h = hashes["motion_acceptance6"]
    f = O.synth_bytes(h["frames"] * h["w"] * h["h"], h["seed"])
    assert sha(f) == h["input_sha256"]
    assert sha(O.motion_gray(f, h["w"], h["h"], h["thr"])) == h["out_sha256"]


def test_gauss_kats():
    # proj/tests/test_motion.cpp:74-117
    for v in (0, 37, 255):
        img = np.full(16 * 12, v, np.uint8)
        np.testing.assert_array_equal(O.gauss5x5(img, 16, 12), img)
    img = np.zeros(21 * 17, np.uint8)
    img[8 * 21 + 10] = 255
    assert O.gauss5x5(img, 21, 17)[8 * 21 + 10] == (255 * 36 + 128) >> 8


def test_median_and_thres_kats():
    img = np.zeros(81, np.uint8)
    img[4 * 9 + 4] = 255
    assert O.median5(img, 9, 9)[4 * 9 + 4] == 0
    prev = np.zeros(25, np.uint8)
    assert O.thres_diff(prev, np.full(25, 32, np.uint8), 5, 5, 32)[0] == 0
    assert O.thres_diff(prev, np.full(25, 33, np.uint8), 5, 5, 32)[0] == 255


def test_rgb_gray_restatement_is_bt601_integer():
    rgb = O.synth_bytes(3 * 1000, 5)
    r, g, b = (rgb[0::3].astype(np.uint32), rgb[1::3].astype(np.uint32), rgb[2::3].astype(np.uint32))
    np.testing.assert_array_equal(O.rgb_to_gray(rgb), ((77 * r + 150 * g + 29 * b + 128) >> 8).astype(np.uint8))
    # gray(RGB) then the pinned gray chain
    rgb = O.synth_bytes(3 * 4 * 40 * 30, 9)
    gray = O.rgb_to_gray(rgb)
    np.testing.assert_array_equal(O.motion_rgb(rgb, 40, 30), O.motion_gray(gray, 40, 30))


def test_channel_slot_walk_fig2():
    # proj/tests/acceptance.cpp:87-137 (criteria [1], [2])
    for r in (1, 2, 3, 4, 8, 16):
        assert O.capacity_tokens(r, True) == 3 * r + 1
        assert O.capacity_tokens(r, False) == 2 * r
    assert [O.write_slot(4, True, p) for p in range(4)] == [1, 5, 9, 1]
    assert [O.read_slot(4, True, p) for p in range(4)] == [0, 4, 8, 0]


def test_compare_samples_semantics():
    w = np.array([1.0, 0.0, 1e-4, 0.0], np.float32)
    g = w.copy()
    assert O.compare_samples(g, w) == (-1, 0.0)
    g[2] += 2e-8  # |err| / max(|w|, 1e-3) = 2e-5
    idx, worst = O.compare_samples(g, w)
    assert idx == 1 and worst > 1e-5


ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@ref_only
def test_oracle_vs_compiled_reference_random_dpd():
    import ctypes as C
    R = O.ref()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rng = np.random.default_rng(0)
    for trial in range(6):
        period = int(rng.choice([1, 3, 8, 9, 10, 64, 257]))
        blocks = int(rng.integers(1, 9))
        sched = rng.integers(0, 1024, size=int(rng.integers(1, 6))).astype(np.uint16)
        x = O.synth_samples(period * blocks, 100 + trial)
        t = O.random_taps(200 + trial)
        want = np.empty_like(x)
        assert R.ref_oracle_dpd(P(x), x.size // 2, P(t), P(sched), sched.size, period, P(want)) == 0
        np.testing.assert_array_equal(bits(O.dpd(x, t, sched, period)), bits(want))


@ref_only
def test_oracle_vs_compiled_reference_motion_sizes():
    import ctypes as C
    R = O.ref()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    for (w, h, n, thr) in [(5, 5, 3, 32), (17, 13, 4, 10), (64, 8, 3, 200)]:
        f = O.synth_bytes(w * h * n, w * h)
        want = np.empty_like(f)
        R.ref_oracle_motion(P(f), n, w, h, thr, P(want))
        np.testing.assert_array_equal(O.motion_gray(f, w, h, thr), want)


@pytest.mark.parametrize("period,T,blocks", [(64, 10, 37), (4, 10, 50), (7, 32, 40), (256, 32, 12), (1, 10, 60)])
def test_dpd_mt_equals_serial(period, T, blocks):
    """The threaded oracle (block ranges, FIR history rebuilt from each
    branch's active stream) is bit-identical to the serial restatement,
    including blocks shorter than T-1 and branches gated off for long runs."""
    x = O.synth_samples(period * blocks, 5 + T)
    taps = O.random_taps(6, T)
    sched = np.array([0x3FF, 0x001, 0x200, 0x000, 0x2A5, 0x100, 0x100, 0x0F0, 0x001, 0x155, 0x300], np.uint16)
    want = O.dpd(x, taps, sched, period)
    for threads in (1, 3, 7):
        np.testing.assert_array_equal(O.dpd_mt(x, taps, sched, period, threads).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("fmt", [1, 3])
def test_motion_mt_equals_serial(fmt):
    w, h, n = 40, 24, 23
    f = O.synth_bytes(n * w * h * fmt, 77)
    want = O.motion_rgb(f, w, h, 32) if fmt == 3 else O.motion_gray(f, w, h, 32)
    for threads in (1, 4, 9):
        np.testing.assert_array_equal(O.motion_mt(f, w, h, fmt, 32, threads=threads), want)
    if fmt == 3:
        halo = O.synth_bytes(w * h * 3, 78)
        np.testing.assert_array_equal(O.motion_mt(f, w, h, 3, 32, prev_rgb=halo, threads=5),
                                      O.motion_rgb(f, w, h, 32, halo))
