"""GPU: the drop-in proven through the REFERENCE's own runtime.

oracle/_ref/dropin_ref (tests/dropin/dropin_ref.cpp, built by
`make -C oracle ref` from the reference's unmodified sources and headers plus
libdf_cuda.so) runs networks through dynflow::run -- the reference's thread-
per-actor runtime -- with GPU actors from libdf_cuda.so in place of the
reference's kernels:
  * motion: gauss/thres/med -> one GPU actor behind dynflow::bulk_kernel_adapter
    (proj/include/dynflow/runtime.hpp:97-108), r = 1 and 4, byte-equal to
    oracle_motion_detection_raw on acceptance [6]'s input;
  * DPD: split/10 branches/adder -> one dynamic GPU actor (its control is the
    reference's check_config), bit-equal to oracle_dpd on acceptance [8] and a
    period-4096 random schedule;
  * a failing C-ABI call inside fire ends run() in ActorFault naming the actor.
The binary is built in the build container (the reference's headers are not
on the GPU box) and travels with the snapshot like the other built .so files.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_ref")

pytestmark = pytest.mark.gpu


def test_gpu_actors_inside_reference_runtime(gpu):
    assert os.path.exists(BIN), f"{BIN} missing: run __graft_entry__.build() in the build container"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = r.stdout.strip().splitlines()
    verdicts = {ln.split()[1]: ln.split()[0] for ln in lines if ln.startswith(("PASS", "FAIL"))}
    assert verdicts == {"motion_r1": "PASS", "motion_r4": "PASS", "dpd_acc8": "PASS", "dpd_p4096": "PASS",
                        "fault": "PASS"}, r.stdout + r.stderr
    assert r.returncode == 0
