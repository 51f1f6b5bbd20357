"""GPU parity: the fused sm_100a motion-detection actor vs the oracle and
the reference's fixtures -- byte-exact.  Pins follow
proj/tests/test_motion.cpp and proj/tests/acceptance.cpp [6], [7]."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def run_gpu(frames, w, h, thr=32, fmt=1, chunk=0, prev=None):
    from paper_1611_03226_b200 import motion
    from paper_1611_03226_b200.device import Buffer
    a = motion.MotionActor(w, h, fmt, thr)
    if prev is not None:
        pb = Buffer.from_array(prev)
        a.set_prev_frame(pb)
    frames = np.ascontiguousarray(frames, np.uint8)
    out = np.empty(frames.size // fmt, np.uint8)
    a.run_host(frames, out, chunk_frames=chunk)
    return out


def assert_frames_equal(got, want, w, h):
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        i = int(bad[0])
        f, r = divmod(i, w * h)
        raise AssertionError(f"{bad.size} bytes differ; first frame {f} row {r // w} col {r % w}: "
                             f"got {got[i]} want {want[i]}")


def test_acceptance6_320x240(gpu, hashes):
    h = hashes["motion_acceptance6"]
    f = O.synth_bytes(h["frames"] * h["w"] * h["h"], h["seed"])
    for chunk in (0, 1, 4):  # token rate r = 1 and 4 per firing (criterion [6])
        out = run_gpu(f, h["w"], h["h"], h["thr"], chunk=chunk)
        assert hashlib.sha256(out.tobytes()).hexdigest() == h["out_sha256"], chunk


def test_reference_fixture_64x48(gpu, small):
    out = run_gpu(small["motion_64x48_in"], 64, 48)
    assert_frames_equal(out, small["motion_64x48_out"], 64, 48)


@pytest.mark.parametrize("thr", [0, 32, 127, 128, 254])
def test_odd_size_and_thresholds(gpu, small, thr):
    out = run_gpu(small["motion_33x29_in"], 33, 29, thr)
    assert_frames_equal(out, small[f"motion_33x29_t{thr}_out"], 33, 29)


@pytest.mark.parametrize("w,h", [(5, 5), (8, 5), (9, 9), (16, 12), (17, 13), (21, 17), (30, 20), (240, 40),
                                 (248, 33), (256, 64), (480, 70), (488, 65), (1280, 72)])
def test_sizes_vs_oracle(gpu, w, h):
    n = 5
    f = O.synth_bytes(n * w * h, w * 1000 + h)
    assert_frames_equal(run_gpu(f, w, h), O.motion_gray(f, w, h), w, h)


@pytest.mark.parametrize("thr", [1, 32, 200, 255])
def test_structured_frames(gpu, thr):
    # Smooth moving pattern: thresholds bite (random noise saturates them).
    w, h, n = 96, 40, 6
    yy, xx = np.mgrid[0:h, 0:w]
    frames = np.stack([((xx * 3 + yy * 2 + 17 * t) % 256) for t in range(n)]).astype(np.uint8)
    frames[2, 10:20, 30:50] = 255
    frames[4, 0:3, :] = 0
    assert_frames_equal(run_gpu(frames, w, h, thr), O.motion_gray(frames, w, h, thr), w, h)


@pytest.mark.parametrize("w,h", [(1280, 720), (64, 48), (33, 29)])
def test_rgb_input(gpu, w, h):
    n = 3
    rgb = O.synth_bytes(n * w * h * 3, 7 + w)
    assert_frames_equal(run_gpu(rgb, w, h, fmt=3), O.motion_rgb(rgb, w, h), w, h)


@pytest.mark.parametrize("w,h,fmt", [(256, 300, 1), (264, 170, 1), (1280, 200, 3), (488, 240, 3), (96, 117, 3)])
def test_interior_bands_vs_oracle(gpu, w, h, fmt):
    # Frames tall enough that most bands take the interior pass (fixed trip
    # count, no row clamps), next to the general pass of the border bands.
    n = 4
    f = O.synth_bytes(n * w * h * fmt, 3 * w + h)
    want = O.motion_rgb(f, w, h) if fmt == 3 else O.motion_gray(f, w, h)
    assert_frames_equal(run_gpu(f, w, h, fmt=fmt), want, w, h)


def test_interior_bands_temporal_chunks_structured(gpu):
    # Structured motion (thresholds bite) over many frames: frame-range
    # warm-up passes (MODE 0) and delay-token passes (MODE 2) in interior bands.
    w, h, n = 512, 264, 41
    yy, xx = np.mgrid[0:h, 0:w]
    frames = np.stack([((xx * 5 + yy * 3 + 11 * t) % 251) for t in range(n)]).astype(np.uint8)
    frames[7, 60:140, 100:300] = 255
    frames[20, 100:101, :] = 0
    want = O.motion_gray(frames.reshape(-1), w, h, 40)
    assert_frames_equal(run_gpu(frames.reshape(-1), w, h, 40), want, w, h)
    for chunk in (3, 17):
        assert_frames_equal(run_gpu(frames.reshape(-1), w, h, 40, chunk=chunk), want, w, h)


@pytest.mark.parametrize("ri", [0, 1, 2])
@pytest.mark.parametrize("w,h,fmt,n,chunk", [(1280, 300, 3, 9, 4), (320, 240, 1, 13, 0), (640, 137, 3, 5, 1),
                                             (96, 40, 3, 6, 2)])
def test_tma_tmem_band_heights(gpu, monkeypatch, ri, w, h, fmt, n, chunk):
    # The TMA/TMEM kernel (rows 16-byte aligned: W*FMT % 16 == 0) at each of
    # its band heights, across firings (delay token) and temporal chunks.
    monkeypatch.setenv("DF_MOTION_M3_R", str(ri))
    f = O.synth_bytes(n * w * h * fmt, 100 * ri + w + h)
    want = O.motion_rgb(f, w, h) if fmt == 3 else O.motion_gray(f, w, h)
    assert_frames_equal(run_gpu(f, w, h, fmt=fmt, chunk=chunk), want, w, h)


def test_kernel_selection(gpu):
    # 16-byte aligned rows take the TMA/TMEM kernel, the rest the
    # register-prefetch kernel: both are exercised by this suite.
    from paper_1611_03226_b200 import motion
    assert motion.MotionActor(1280, 720, motion.RGB).kernel_name == "motion_m3_kernel"
    assert motion.MotionActor(3840, 2160, motion.RGB).kernel_name == "motion_m3_kernel"
    assert motion.MotionActor(320, 240, motion.GRAY).kernel_name == "motion_m3_kernel"
    assert motion.MotionActor(488, 65, motion.RGB).kernel_name == "motion_fused_kernel"
    assert motion.MotionActor(33, 29, motion.GRAY).kernel_name == "motion_fused_kernel"


@pytest.mark.parametrize("h", [5, 6, 7, 28, 29, 30, 34, 35, 39, 40, 41, 44, 49, 50, 53, 54, 55, 59, 60, 61, 78, 79,
                               108, 109, 113, 115])
@pytest.mark.parametrize("ri", [0, 1, 2])
def test_tma_tmem_heights_near_band_edges(gpu, monkeypatch, ri, h):
    # Frame heights around the band heights (gray, 16 px per lane: 29/34/39;
    # RGB: 39/44/49): last bands of 1..R rows, bands entirely in the border,
    # interior/general band mixes.
    monkeypatch.setenv("DF_MOTION_M3_R", str(ri))
    w, n = 256, 3
    f = O.synth_bytes(n * w * h, 1000 * ri + h)
    assert_frames_equal(run_gpu(f, w, h, chunk=2), O.motion_gray(f, w, h), w, h)


@pytest.mark.parametrize("w", [16, 32, 464, 480, 496, 960, 976, 1296])
@pytest.mark.parametrize("h", [5, 40, 79])
def test_gray_wide_lane_tiles(gpu, w, h):
    # Gray runs the TMA/TMEM kernel at 16 px per lane (480-px tiles, 12-warp
    # CTAs): frames narrower than a tile, exactly one or two tiles, a last
    # tile holding a single 16-px lane, and the frame edge inside a lane word.
    from paper_1611_03226_b200 import motion
    assert motion.MotionActor(w, h, motion.GRAY).kernel_name == "motion_m3_kernel"
    n = 4
    f = O.synth_bytes(n * w * h, 7 * w + h)
    assert_frames_equal(run_gpu(f, w, h, chunk=3), O.motion_gray(f, w, h), w, h)


@pytest.mark.parametrize("thr", [0, 1, 127, 128, 254, 255])
def test_tma_tmem_gray_thresholds_structured(gpu, thr):
    w, h, n = 512, 140, 7
    yy, xx = np.mgrid[0:h, 0:w]
    frames = np.stack([((xx * 3 + yy + 13 * t) % 256) for t in range(n)]).astype(np.uint8)
    frames[3, 20:90, 100:400] = 255
    frames[5, :, 0:2] = 0
    frames[5, :, w - 2:] = 255
    f = frames.reshape(-1)
    assert_frames_equal(run_gpu(f, w, h, thr), O.motion_gray(f, w, h, thr), w, h)


@pytest.mark.parametrize("thr", [0, 1, 127, 128, 254, 255])
def test_tma_tmem_thresholds_structured(gpu, thr):
    w, h, n = 512, 140, 7
    yy, xx = np.mgrid[0:h, 0:w]
    rgb = np.stack([np.stack([(xx * 3 + yy + 13 * t) % 256, (xx + 2 * yy + 7 * t) % 256,
                              (5 * xx + yy * 3 + 29 * t) % 256], -1) for t in range(n)]).astype(np.uint8)
    rgb[3, 20:90, 100:400] = 255
    f = rgb.reshape(-1)
    assert_frames_equal(run_gpu(f, w, h, thr, fmt=3), O.motion_rgb(f, w, h, thr), w, h)


def test_many_frames_temporal_chunks(gpu):
    # Enough frames that the kernel splits the firing into frame ranges,
    # each recomputing gauss(f0 - 1) on chip.
    w, h, n = 320, 96, 97
    f = O.synth_bytes(n * w * h, 42)
    assert_frames_equal(run_gpu(f, w, h), O.motion_gray(f, w, h), w, h)


def test_chunked_firings_carry_delay_token(gpu):
    w, h, n = 64, 40, 23
    f = O.synth_bytes(n * w * h, 17)
    want = O.motion_gray(f, w, h)
    for chunk in (1, 2, 5, 22):
        assert_frames_equal(run_gpu(f, w, h, chunk=chunk), want, w, h)


def test_frame_range_shard_with_halo(gpu):
    # Shard [f0, f1) with the one-frame halo f0-1 as the delay token equals
    # the corresponding slice of the full run (the multi-GPU decomposition).
    w, h, n = 96, 48, 12
    rgb = O.synth_bytes(n * w * h * 3, 99)
    full = O.motion_rgb(rgb, w, h)
    fsz = w * h
    for f0, f1 in [(0, 5), (5, 12), (7, 8)]:
        prev = rgb[(f0 - 1) * fsz * 3: f0 * fsz * 3] if f0 > 0 else None
        got = run_gpu(rgb[f0 * fsz * 3: f1 * fsz * 3], w, h, fmt=3, prev=prev)
        assert_frames_equal(got, full[f0 * fsz: f1 * fsz], w, h)


@pytest.mark.parametrize("w,h,n", [(96, 48, 12), (1280, 72, 9), (160, 130, 40), (44, 30, 6), (250, 61, 17)])
def test_fire_halo_equals_shard_of_full_run(gpu, w, h, n):
    """df_motion_fire_halo (gauss of the halo frame computed in-kernel by the
    shard's first temporal chunk) == the same shard of the full run, for M3
    widths (96, 1280, 160: W*3 % 16 == 0) and fallback widths (44, 250)."""
    from paper_1611_03226_b200 import device, motion
    rgb = O.synth_bytes(n * w * h * 3, 1000 + w)
    full = O.motion_rgb(rgb, w, h)
    fb = w * h * 3
    f0, f1 = n // 3, n - 2
    a = motion.MotionActor(w, h, motion.RGB, 32)
    inp = device.Buffer.from_array(rgb[f0 * fb:])
    halo = device.Buffer.from_array(rgb[(f0 - 1) * fb:f0 * fb])
    out = device.Buffer((n - f0) * w * h)
    a.fire_halo(halo, inp, out, f1 - f0)
    # ... and the delay token it leaves carries into the next firing
    a.fire(inp, out, n - f1, in_offset=(f1 - f0) * fb, out_offset=(f1 - f0) * w * h)
    assert_frames_equal(out.download(np.uint8), full[f0 * w * h:], w, h)


def test_first_frame_against_black(gpu):
    # proj/tests/test_motion.cpp:183-192
    f = np.full(8 * 8, 200, np.uint8)
    assert (run_gpu(f, 8, 8) == 255).all()


def test_delay_dependency_acceptance7(gpu):
    # proj/tests/acceptance.cpp:344-373
    w, h, n = 320, 240, 64
    size = w * h
    f = O.synth_bytes(n * size, 707)
    base = run_gpu(f, w, h)
    rng = np.random.default_rng(708)
    for _ in range(3):
        j = int(rng.integers(0, n))
        p = f.copy().reshape(n, h, w)
        p[j, 40:56, 40:56] = 0
        out = run_gpu(p.reshape(-1), w, h)
        for fr in range(n):
            differs = not np.array_equal(out[fr * size:(fr + 1) * size], base[fr * size:(fr + 1) * size])
            if fr in (j, j + 1):
                if fr == j:
                    assert differs
            else:
                assert not differs, (j, fr)


def test_stage_kernels(gpu):
    from paper_1611_03226_b200 import motion
    w, h = 33, 29
    img = O.synth_bytes(w * h, 1)
    np.testing.assert_array_equal(motion.gauss5x5(img, w, h), O.gauss5x5(img, w, h))
    np.testing.assert_array_equal(motion.median5(img, w, h), O.median5(img, w, h))
    prev = O.synth_bytes(w * h, 2)
    np.testing.assert_array_equal(motion.thres_diff(prev, img, w, h, 32), O.thres_diff(prev, img, w, h, 32))
    rgb = O.synth_bytes(3 * 1000, 3)
    np.testing.assert_array_equal(motion.rgb_to_gray(rgb), O.rgb_to_gray(rgb))


def test_channel_bound_firing_with_delay_channel(gpu):
    """Fig. 2 on device: a rate-1 self-loop delay channel carries gauss of
    the last frame between firings (proj/tests/test_runtime.cpp:401-429)."""
    import ctypes as C
    from paper_1611_03226_b200 import motion
    from paper_1611_03226_b200._lib import call
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Stream
    w, h, r, rounds = 64, 48, 4, 7  # 7 firings walk the delay slots through 2+ cycles
    f = O.synth_bytes(r * rounds * w * h * 3, 5)
    s = Stream()
    cin = DeviceChannel(w * h * 3, r)
    cout = DeviceChannel(w * h, r)
    delay = DeviceChannel(w * h, 1, has_delay=True)
    a = motion.MotionActor(w, h, motion.RGB)
    got = np.empty(r * rounds * w * h, np.uint8)
    for k in range(rounds):
        wr = cin.write_start(r)
        blk = np.ascontiguousarray(f[k * r * w * h * 3:(k + 1) * r * w * h * 3])
        call("df_memcpy_h2d", C.c_void_p(wr.dptr), blk.ctypes.data_as(C.c_void_p), blk.nbytes, s.handle)
        cin.write_end(wr, s)
        a.fire_channels(cin, delay, cout, s)
        rd = cout.read_start(r)
        part = np.empty(r * w * h, np.uint8)
        call("df_memcpy_d2h", part.ctypes.data_as(C.c_void_p), C.c_void_p(rd.dptr), part.nbytes, s.handle)
        cout.read_end(rd, s)
        s.synchronize()
        got[k * r * w * h:(k + 1) * r * w * h] = part
    for ch in (cin, cout, delay):
        ch.check()
    st = delay.stats()
    assert st.tokens_written == rounds and st.tokens_read == rounds and st.tokens_available == 1
    assert st.write_phase == rounds % 3 and st.read_phase == rounds % 3
    assert_frames_equal(got, O.motion_rgb(f, w, h), w, h)


def test_empty_firings_keep_the_delay_token(gpu):
    """Zero frames (the reference's network with frames = 0 fires nothing,
    motion.cpp:104) is a no-op at every entry point: a zero-frame fire or
    run_host between two runs changes neither the output nor the delay
    token the next firing diffs against."""
    from paper_1611_03226_b200 import motion
    from paper_1611_03226_b200.device import Buffer
    w, h, n = 96, 40, 6
    f = O.synth_bytes(n * w * h, 77)
    want = O.motion_gray(f, w, h, 32)
    a = motion.MotionActor(w, h, motion.GRAY, 32)
    got = np.empty(n * w * h, np.uint8)
    a.run_host(f[: 3 * w * h], got[: 3 * w * h])
    a.run_host(f[:0], got[:0])
    scratch = Buffer(w * h)
    a.fire(scratch, scratch, 0)
    a.run_host(f[3 * w * h:], got[3 * w * h:])
    assert_frames_equal(got, want, w, h)
