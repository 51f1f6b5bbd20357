"""GPU: bench.py's N > 1 path end to end -- torchrun with 2 or 8 ranks
sharing cuda:0 (gloo for setup and timing reductions; NCCL refuses two ranks
on one GPU), the IPC halo transport, frame-range / block-range shards,
max-over-rank timing -- prints one well-formed JSON line from rank 0 with
n_gpus = N.  The 8-rank runs are the driver's scaling configurations
(configs[3] motion 4K, configs[4] DPD 10 x 32) at their per-GPU sizes.
Numbers from these runs are not bench values (the ranks time-share one GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,ranks", [("motion720", 2), ("dpd3", 2), ("motion720", 8), ("motion4k", 8),
                                            ("dpd5", 8)])
def test_bench_multi_rank(gpu, workload, ranks):
    env = dict(os.environ, DF_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(ranks),
           "--workload", workload, "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == ranks and d["steps"] == 3 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert "CUDA IPC" in d["config"]["parallelism"]
