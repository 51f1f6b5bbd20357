"""GPU, BASELINE full sizes (the bench's own configs): the oracle is too slow
for whole streams, so parity at full size is shown by size-independent
properties plus oracle checks of sampled frames / blocks (each computed
from exactly the inputs it depends on):

* motion 1280x720 RGB x 300 and 3840x2160 RGB x 40: one firing == the same
  frames in uneven firings (delay token carried; different M3 plans), and
  sampled masks == the oracle on (frame f-2 as halo, f-1, f);
* DPD-5 (10 branches x 32 taps, 2^27 samples) and DPD-3 (ramp, 4096-sample
  blocks, 2^26): one batch == two batches (FirState carried), the leading
  2^20 samples and sampled blocks == the oracle on the blocks they depend
  on (history reaches back at most one block for DPD-5, 10 for the ramp).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _motion_host(rgb, w, h, splits):
    from paper_1611_03226_b200 import motion
    a = motion.MotionActor(w, h, motion.RGB, 32)
    fb = w * h * 3
    out = np.empty(rgb.size // 3, np.uint8)
    f0 = 0
    for n in splits:
        a.run_host(rgb[f0 * fb:(f0 + n) * fb], out[f0 * w * h:(f0 + n) * w * h])
        f0 += n
    return out


@pytest.mark.parametrize("w,h,n,splits", [(1280, 720, 300, (97, 103, 100)), (3840, 2160, 40, (13, 27))])
def test_motion_full_size(gpu, w, h, n, splits):
    fb, px = w * h * 3, w * h
    rgb = O.synth_bytes(n * fb, 20240 + w)
    whole = _motion_host(rgb, w, h, (n,))
    assert np.array_equal(whole, _motion_host(rgb, w, h, splits)), "firing split changed the masks"
    for f in (0, 1, splits[0], n // 2 + 1, n - 1):
        if f == 0:
            want = O.motion_rgb(rgb[:fb], w, h, 32)
        elif f == 1:
            want = O.motion_rgb(rgb[:2 * fb], w, h, 32)[px:]
        else:
            want = O.motion_rgb(rgb[(f - 1) * fb:(f + 1) * fb], w, h, 32, rgb[(f - 2) * fb:(f - 1) * fb])[px:]
        got = whole[f * px:(f + 1) * px]
        assert np.array_equal(got, want), f"frame {f}: {(got != want).sum()} bytes differ"


def _dpd_host(x, taps, sched, period, splits):
    from paper_1611_03226_b200 import dpd
    a = dpd.DpdActor(period, taps)
    out = np.empty_like(x)
    s0 = 0
    for nb in splits:
        lo, hi = 2 * s0 * period, 2 * (s0 + nb) * period
        # the schedule cycles per block from the stream start (dpd.cpp:208);
        # run_host continues it from the blocks earlier calls fired
        a.run_host(x[lo:hi], out[lo:hi], sched)
        s0 += nb
    a.check()
    return out


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("name", ["dpd5", "dpd3"])
def test_dpd_full_size(gpu, name):
    if name == "dpd5":
        samples, period, T = 1 << 27, 65536, 32
        sched = np.array([0x3FF], np.uint16)
        back = 1
    else:
        samples, period, T = 1 << 26, 4096, 10
        sched = np.array([(1 << (1 + i % 10)) - 1 for i in range(10)], np.uint16)
        back = 10
    blocks = samples // period
    x = O.synth_samples(samples, 8080 + T)
    taps = O.random_taps(8081, T)
    whole = _dpd_host(x, taps, sched, period, (blocks,))
    split = _dpd_host(x, taps, sched, period, (blocks // 3, blocks - blocks // 3))
    assert np.array_equal(_bits(whole), _bits(split)), "batch split changed the output"
    lead = 1 << 20
    assert np.array_equal(_bits(whole[:2 * lead]), _bits(O.dpd(x[:2 * lead], taps, sched, period)))
    for k in (blocks // 3, blocks // 2 + 7, blocks - 1):
        k0 = k - back
        seg = O.dpd(x[2 * k0 * period:2 * (k + 1) * period], taps, np.roll(sched, -(k0 % len(sched))), period)
        got = whole[2 * k * period:2 * (k + 1) * period]
        assert np.array_equal(_bits(got), _bits(seg[2 * back * period:])), f"block {k} differs"
