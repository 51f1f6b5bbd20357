"""`verify` front end: runs the device network and the oracle on identical
input and reports PASS or FAIL with first-divergence diagnostics.

Mirrors the reference's `cmd_verify` (proj/src/bench.cpp:443-490) and its
CLI defaults (proj/include/dynflow/bench.hpp:19-41): synthetic input from
the seed unless --input names a raw file (motion: concatenated W*H gray
frames; dpd: interleaved float re,im pairs), taps random_taps(seed) and
schedule random_schedule(16, seed) (bench.cpp:227-262), the DPD stream
padded to whole periods, motion compared byte-exact (compare_frames,
bench.cpp:288-305), DPD per-sample relative error 1e-5 against a 1e-3
floor (compare_samples, bench.cpp:307-326).  Same output lines (human or
--porcelain) and exit codes: 0 PASS, 1 FAIL, 2 configuration error.

It is a checker, so it lives with the tests: the oracle is test
infrastructure and the product path never imports it.  The device side
is the drop-in network run (`dfh_motion_run` / `dfh_dpd_run` through
host_api), the same call `cmd_motion` / `cmd_dpd` would make.

    python tests/verify_cli.py --app motion --width 320 --height 240 --frames 64 --seed 606
    python tests/verify_cli.py --app dpd --samples 1048576 --period 65536 --porcelain
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402

EXIT_OK, EXIT_VERIFY_FAILED, EXIT_CONFIG_ERROR = 0, 1, 2  # bench.hpp:39-41


class ConfigError(Exception):
    pass


def compare_frames(got: np.ndarray, want: np.ndarray, frame_size: int):
    """bench.cpp:288-305: (frame index, detail) of the first differing byte, or None."""
    if got.size != want.size:
        return 0, f"output size {got.size} != {want.size}"
    bad = np.flatnonzero(got != want)
    if bad.size == 0:
        return None
    i = int(bad[0])
    return i // frame_size, f"frame {i // frame_size} byte {i % frame_size}: got {int(got[i])}, want {int(want[i])}"


def compare_samples(got: np.ndarray, want: np.ndarray):
    """bench.cpp:307-326 via the oracle's restatement: (sample index, detail) or None."""
    if got.size != want.size:
        return 0, f"output size {got.size // 2} != {want.size // 2}"
    idx, _ = O.compare_samples(got, want, 1e-5)
    if idx < 0:
        return None
    g, w = got.reshape(-1, 2)[idx], want.reshape(-1, 2)[idx]
    return idx, f"sample {idx}: got ({g[0]:.9g},{g[1]:.9g}), want ({w[0]:.9g},{w[1]:.9g})"


def load_motion_input(a):
    """bench.cpp:173-204 (raw gray frames or synth_frames(frames, W, H, seed))."""
    size = a.width * a.height
    if not a.input:
        return O.synth_bytes(a.frames * size, a.seed), a.frames
    raw = np.fromfile(a.input, np.uint8)
    if raw.size == 0 or raw.size % size:
        raise ConfigError(f"'{a.input}' is not a multiple of {size}-byte frames")
    frames = raw.size // size
    if 0 < a.frames < frames:
        frames = a.frames
    return raw[:frames * size], frames


def load_dpd_setup(a):
    """bench.cpp:227-262: (padded input, user-visible samples, taps, schedule)."""
    taps = O.random_taps(a.seed)
    schedule = O.random_schedule(16, a.seed)
    if not a.input:
        samples = a.samples
        x = O.synth_samples(samples, a.seed)
    else:
        raw = np.fromfile(a.input, np.uint8)
        if raw.size == 0 or raw.size % 8:
            raise ConfigError(f"'{a.input}' is not interleaved float re,im pairs")
        samples = raw.size // 8
        if 0 < a.samples < samples:
            samples = a.samples
        x = raw[:samples * 8].view(np.float32).copy()
    if samples == 0:
        raise ConfigError("no samples to process")
    padded = (samples + a.period - 1) // a.period * a.period
    x = np.concatenate([x, np.zeros(2 * (padded - samples), np.float32)])
    return x, samples, taps, schedule


def verify(a, out=sys.stdout) -> int:
    from paper_1611_03226_b200 import host_api
    try:
        if a.app == "motion":
            frames_in, frames = load_motion_input(a)
            if frames % a.rate:
                raise ConfigError("frame count is not a multiple of the token rate")
            got, _, _ = host_api.motion_run(frames_in, a.width, a.height, fmt=1, threshold=a.threshold,
                                            rate=a.rate, device=a.device)
            want = O.motion_gray(frames_in, a.width, a.height, a.threshold)
            div = compare_frames(got, want, a.width * a.height)
        else:
            x, _, taps, schedule = load_dpd_setup(a)
            got, _, _ = host_api.dpd_run(x, taps, schedule, a.period, device=a.device)
            want = O.dpd(x, taps, schedule, a.period)
            div = compare_samples(got, want)
    except (ConfigError, ValueError, host_api.HostRunError) as e:
        if a.porcelain:
            print(f"error={e}", file=out)
        else:
            print(f"error: {e}", file=out)
        return EXIT_CONFIG_ERROR
    verdict = "FAIL" if div else "PASS"
    if a.porcelain:
        print(f"app={a.app}\nseed={a.seed}\nverify={verdict}", file=out)
        if div:
            print(f"divergence_index={div[0]}\ndivergence={div[1]}", file=out)
    else:
        print(f"verify {a.app} (seed {a.seed}): {verdict}", file=out)
        if div:
            print(f"first divergence: {div[1]}", file=out)
    return EXIT_VERIFY_FAILED if div else EXIT_OK


def parser():
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--app", choices=["motion", "dpd"], default="motion")
    p.add_argument("--input", default="")
    p.add_argument("--frames", type=int, default=64)
    p.add_argument("--samples", type=int, default=1 << 20)
    p.add_argument("--rate", type=int, default=1)
    p.add_argument("--width", type=int, default=320)
    p.add_argument("--height", type=int, default=240)
    p.add_argument("--threshold", type=int, default=32)
    p.add_argument("--period", type=int, default=65536)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--porcelain", action="store_true")
    return p


if __name__ == "__main__":
    sys.exit(verify(parser().parse_args()))
