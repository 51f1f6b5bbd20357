"""GPU, BASELINE full sizes (the bench's own configs), WHOLE-output parity:
every byte / float word of the GPU output against the oracle on the same
stream.  The oracle runs in parallel over frame / block ranges
(oracle.motion_mt / dpd_mt: each range starts from exactly the state the
serial run has there -- the previous frame's gauss, each branch's FIR
history from its active stream -- and tests/test_oracle.py pins them
bit-identical to the serial restatement).

* motion 1280x720 RGB x 300 (configs[1]) and 3840x2160 RGB x 40 per GPU
  (configs[3]): byte-exact, in one firing and in uneven firings (delay
  token carried across firings; different M3 plans);
* DPD-1 exactly as benched (first_n(2), 2^20, period 65536, configs[0]),
  DPD-3 (ramp 1->10 branches, 4096-sample blocks, 2^26, configs[2]) and
  DPD-5 (10 branches x 32 taps, 2^27 per GPU, configs[4]): bit-exact, in one
  batch and in two (FirState and schedule position carried).
Reference comparators: proj/src/bench.cpp:288-326.
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
    rgb = O.synth_bytes(n * w * h * 3, 20240 + w)
    want = O.motion_mt(rgb, w, h, 3, 32)
    whole = _motion_host(rgb, w, h, (n,))
    bad = np.nonzero(whole != want)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first in frame {bad[0] // (w * h)}"
    split = _motion_host(rgb, w, h, splits)
    assert np.array_equal(split, want), "uneven firings changed the masks"


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


@pytest.mark.parametrize("name", ["dpd1", "dpd3", "dpd5"])
def test_dpd_full_size(gpu, name):
    if name == "dpd1":  # bench.py dpd1: first_n(2)
        samples, period, T = 1 << 20, 65536, 10
        sched = np.array([0x003], np.uint16)
    elif name == "dpd3":  # ramp: block i -> first_n(1 + i % 10)
        samples, period, T = 1 << 26, 4096, 10
        sched = np.array([(1 << (1 + i % 10)) - 1 for i in range(10)], np.uint16)
    else:  # all ten branches, 32 taps
        samples, period, T = 1 << 27, 65536, 32
        sched = np.array([0x3FF], np.uint16)
    blocks = samples // period
    x = O.synth_samples(samples, 8080 + T)
    taps = O.random_taps(8081, T)
    want = O.dpd_mt(x, taps, sched, period)
    whole = _dpd_host(x, taps, sched, period, (blocks,))
    bad = np.nonzero(_bits(whole) != _bits(want))[0]
    assert bad.size == 0, f"{bad.size} float words differ, first at sample {bad[0] // 2}"
    idx, worst = O.compare_samples(whole, want)
    assert idx < 0, worst
    split = _dpd_host(x, taps, sched, period, (blocks // 3, blocks - blocks // 3))
    assert np.array_equal(_bits(split), _bits(want)), "batch split changed the output"
