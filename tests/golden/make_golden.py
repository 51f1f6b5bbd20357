"""Generates tests/golden/* from the UNMODIFIED reference compiled by
oracle/Makefile (oracle/_ref/libdynflow_ref.so, built from
/root/reference/proj/src).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Small cases are stored raw (npz); large acceptance cases as SHA-256 of the
reference output bytes plus the generating seeds.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

R = O.ref()
P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731


def ref_samples(n, seed):
    a = np.empty(2 * n, np.float32)
    R.ref_synth_samples(n, seed, P(a))
    return a


def ref_taps(seed):
    t = np.empty(200, np.float32)
    R.ref_random_taps(seed, P(t))
    return t.reshape(10, 10, 2)


def ref_sched(n, seed):
    s = np.empty(n, np.uint16)
    R.ref_random_schedule(n, seed, P(s))
    return s


def ref_dpd(x, taps, sched, period):
    out = np.empty_like(x)
    rc = R.ref_oracle_dpd(P(x), x.size // 2, P(np.ascontiguousarray(taps)), P(sched), sched.size, period, P(out))
    assert rc == 0
    return out


def ref_frames(frames, w, h, seed):
    f = np.empty(frames * w * h, np.uint8)
    R.ref_synth_frames(frames, w, h, seed, P(f))
    return f


def ref_motion(f, frames, w, h, thr=32):
    out = np.empty_like(f)
    R.ref_oracle_motion(P(f), frames, w, h, thr, P(out))
    return out


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


small = {}
# DPD: reference test pins (proj/tests/test_dpd.cpp:390-408, :457-496) and
# short periods that exercise fir10's chained state (:159-177).
cases = {
    "net_p256_s41": (256, 8, 41, (5, 42), 43),
    "gating_p64": (64, 4, 61, None, 62),
    "short_p4": (4, 16, 80, (5, 3), 10),
    "counts_p16": (16, 6, 51, (3, 52), 53),
}
for name, (period, blocks, tseed, sched_spec, iseed) in cases.items():
    taps = ref_taps(tseed)
    if sched_spec is None:
        sched = np.array([0x3FF, 0x3FF & ~(1 << 4), 0x3F, 0b0000001011], np.uint16)
    else:
        sched = ref_sched(*sched_spec)
    x = ref_samples(period * blocks, iseed)
    small[f"dpd_{name}_in"] = x
    small[f"dpd_{name}_taps"] = taps
    small[f"dpd_{name}_sched"] = sched
    small[f"dpd_{name}_period"] = np.array([period])
    small[f"dpd_{name}_out"] = ref_dpd(x, taps, sched, period)
# single-branch masks (oracle accepts them; the network does not)
x = ref_samples(64 * 10, 7)
t = ref_taps(9)
for k in (1, 2, 10):
    s = np.array([(1 << k) - 1], np.uint16)
    small[f"dpd_k{k}_out"] = ref_dpd(x, t, s, 64)
small["dpd_k_in"], small["dpd_k_taps"] = x, t
# motion: proj/tests/test_motion.cpp:194-217
f = ref_frames(16, 64, 48, 2024)
small["motion_64x48_in"] = f
small["motion_64x48_out"] = ref_motion(f, 16, 64, 48)
f = ref_frames(6, 33, 29, 3)
small["motion_33x29_in"] = f
for thr in (0, 32, 127, 128, 254):
    small[f"motion_33x29_t{thr}_out"] = ref_motion(f, 6, 33, 29, thr)
np.savez_compressed(os.path.join(HERE, "small.npz"), **small)

big = {}
# acceptance [8]: 2^20 samples, period 65536, taps 808, schedule(16, 809), input 810
x = ref_samples(1 << 20, 810)
big["dpd_acceptance8"] = {"samples": 1 << 20, "period": 65536, "taps_seed": 808, "sched": [16, 809],
                          "input_seed": 810, "input_sha256": sha(x),
                          "out_sha256": sha(ref_dpd(x, ref_taps(808), ref_sched(16, 809), 65536))}
# 2^20 at period 4096 with a random 2..10 schedule
y = ref_dpd(x, ref_taps(1), ref_sched(16, 1), 4096)
big["dpd_p4096_random"] = {"samples": 1 << 20, "period": 4096, "taps_seed": 1, "sched": [16, 1],
                           "input_seed": 810, "out_sha256": sha(y)}
# acceptance [6]: 64 frames 320x240 seed 606
f = ref_frames(64, 320, 240, 606)
big["motion_acceptance6"] = {"frames": 64, "w": 320, "h": 240, "seed": 606, "thr": 32,
                             "input_sha256": sha(f), "out_sha256": sha(ref_motion(f, 64, 320, 240))}
# generator stream pins
big["generators"] = {"taps808": ref_taps(808).reshape(-1).tolist(), "sched16_809": ref_sched(16, 809).tolist(),
                     "frames_606_first64": ref_frames(1, 320, 240, 606)[:64].tolist()}
big["mem_totals"] = {"motion_320x240_r1": int(R.ref_mem_total(1, 320, 240, 1, 65536)),
                     "dpd_p65536": int(R.ref_mem_total(0, 320, 240, 1, 65536))}
with open(os.path.join(HERE, "reference_hashes.json"), "w") as fh:
    json.dump(big, fh, indent=1)
print("wrote", sorted(small)[:3], "...", len(small), "arrays;", list(big))
