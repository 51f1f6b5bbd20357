"""The `verify` front end (tests/verify_cli.py), after the reference's
cmd_verify (proj/src/bench.cpp:443-490) and its CLI tests' PASS/FAIL lines."""
import io
import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import verify_cli as V  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1611_03226_b200 import host_api  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def args(*argv):
    return V.parser().parse_args(list(argv))


def test_compare_frames_first_divergence():
    want = np.zeros(3 * 12, np.uint8)
    got = want.copy()
    assert V.compare_frames(got, want, 12) is None
    got[2 * 12 + 5] = 255
    got[2 * 12 + 7] = 255
    assert V.compare_frames(got, want, 12) == (2, "frame 2 byte 5: got 255, want 0")
    assert V.compare_frames(got[:12], want, 12)[1] == "output size 12 != 36"


def test_compare_samples_tolerance():
    want = O.synth_samples(64, 3)
    got = want.copy()
    assert V.compare_samples(got, want) is None
    got[2 * 9] *= 1 + 1e-6  # within 1e-5
    assert V.compare_samples(got, want) is None
    got[2 * 11 + 1] += 0.5
    idx, detail = V.compare_samples(got, want)
    assert idx == 11 and detail.startswith("sample 11: got (")


def test_dpd_setup_pads_to_whole_periods():
    x, samples, taps, schedule = V.load_dpd_setup(args("--app", "dpd", "--samples", "5000", "--period", "4096"))
    assert samples == 5000 and x.size == 2 * 8192
    assert np.array_equal(x[:10000], O.synth_samples(5000, 1)) and not x[10000:].any()
    assert taps.shape == (10, 10, 2) and schedule.size == 16


def test_config_errors_exit_2(tmp_path):
    bad = tmp_path / "frames.raw"
    bad.write_bytes(b"\0" * 1000)  # not a multiple of 320 x 240
    out = io.StringIO()
    assert V.verify(args("--input", str(bad)), out) == V.EXIT_CONFIG_ERROR
    assert "not a multiple of 76800-byte frames" in out.getvalue()
    out = io.StringIO()
    assert V.verify(args("--frames", "10", "--rate", "4", "--porcelain"), out) == V.EXIT_CONFIG_ERROR
    assert out.getvalue().startswith("error=frame count is not a multiple of the token rate")


def test_fail_reports_first_divergence(monkeypatch):
    """FAIL path with a device result corrupted at frame 3 (no GPU needed)."""
    W, H = 32, 16

    def fake_motion_run(frames, width, height, fmt, threshold, rate, device):
        m = O.motion_gray(frames, width, height, threshold)
        m[3 * W * H + 40] ^= 0xFF
        return m, 0.0, 0

    monkeypatch.setattr(host_api, "motion_run", fake_motion_run)
    out = io.StringIO()
    rc = V.verify(args("--width", str(W), "--height", str(H), "--frames", "8", "--porcelain"), out)
    assert rc == V.EXIT_VERIFY_FAILED
    lines = out.getvalue().splitlines()
    assert lines[:3] == ["app=motion", "seed=1", "verify=FAIL"]
    assert lines[3] == "divergence_index=3" and lines[4].startswith("divergence=frame 3 byte 40: got ")


@pytest.mark.gpu
@pytest.mark.parametrize("rate", [1, 4])
def test_motion_verify_passes_acceptance6(gpu, rate):
    """acceptance [6]: 64 frames at 320x240, seed 606, r in {1, 4} (proj/tests/acceptance.cpp:328-341)."""
    out = io.StringIO()
    assert V.verify(args("--frames", "64", "--seed", "606", "--rate", str(rate)), out) == V.EXIT_OK
    assert out.getvalue() == "verify motion (seed 606): PASS\n"


@pytest.mark.gpu
def test_dpd_verify_passes_cli(gpu):
    """The CLI as a process, porcelain output; ragged sample count (padded tail)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "verify_cli.py"), "--app", "dpd", "--samples",
                        str((1 << 18) + 123), "--period", "4096", "--seed", "43", "--porcelain"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout == "app=dpd\nseed=43\nverify=PASS\n"


def test_dpd_fail_reports_first_divergent_sample(monkeypatch):
    """DPD FAIL path: a device result off by 1e-3 relative at sample 4100 (no GPU needed)."""

    def fake_dpd_run(x, taps, schedule, period, device):
        y = O.dpd(x, taps, schedule, period)
        y[2 * 4100] = y[2 * 4100] * (1 + 1e-3) + 1e-3
        return y, 0.0, 0

    monkeypatch.setattr(host_api, "dpd_run", fake_dpd_run)
    out = io.StringIO()
    rc = V.verify(args("--app", "dpd", "--samples", "8192", "--period", "1024", "--seed", "5"), out)
    assert rc == V.EXIT_VERIFY_FAILED
    lines = out.getvalue().splitlines()
    assert lines[0] == "verify dpd (seed 5): FAIL"
    assert lines[1].startswith("first divergence: sample 4100: got (")
