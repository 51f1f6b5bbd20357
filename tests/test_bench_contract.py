"""CPU: bench.py's workload table and algorithmic-work formulas match the
BASELINE configs and SURVEY 8(d) (no GPU needed)."""
import json
import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workloads_cover_baseline_configs():
    cfg = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert len(cfg) == 5
    w = bench.WORKLOADS
    assert w["dpd1"][1]["samples"] == 1 << 20 and w["dpd1"][1]["T"] == 10 and w["dpd1"][1]["sched"] == "first2"
    assert w["motion720"][1]["w"] == 1280 and w["motion720"][1]["h"] == 720 and w["motion720"][1]["frames"] == 300
    assert w["motion720"][1]["fmt"] == 3  # RGB, as configs[1] states
    assert w["dpd3"][1]["period"] == 4096 and w["dpd3"][1]["sched"] == "ramp"
    assert w["motion4k"][1]["w"] == 3840 and w["motion4k"][1]["frames"] * 8 == 320
    assert w["dpd5"][1]["T"] == 32 and w["dpd5"][1]["samples"] * 8 == 1 << 30


@pytest.mark.parametrize("name,want", [("dpd1", 173), ("dpd3", 470), ("dpd5", 2613)])
def test_dpd_flops_per_sample_matches_survey(name, want):
    p = bench.WORKLOADS[name][1]
    sched = bench.dpd_schedule(p["sched"], p["samples"] // p["period"])
    assert abs(bench.dpd_flops_per_sample(sched, p["T"]) - want) < 1.0


def test_ramp_schedule_is_1_to_10_branches():
    s = bench.dpd_schedule("ramp", 20)
    assert [bin(int(m)).count("1") for m in s] == list(range(1, 11))
    assert all(int(m) == (1 << bin(int(m)).count("1")) - 1 for m in s)  # first_n(k)


def test_default_run_is_n1_motion720():
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--gpus", type=int, default=1)' in src
    assert 'ap.add_argument("--workload", default="motion720"' in src
    assert "args.warmup = max(args.warmup, 3)" in src


def test_l2_rule_every_workload_flushes_or_exceeds_l2():
    """Timing rule: between timed steps either flush L2 or use data larger
    than L2 (126 MB).  DPD workloads whose in+out is below L2_FLUSH_BYTES
    rotate over a pool of batches larger than L2 (every step reads a cold
    batch); every other workload's input alone exceeds L2."""
    l2 = 126e6
    assert bench.L2_FLUSH_BYTES > l2
    src = open(bench.__file__).read()
    assert "R = max(1, -(-L2_FLUSH_BYTES // (16 * N)))" in src
    for name, (kind, p) in bench.WORKLOADS.items():
        if kind == "dpd":
            pooled = 16 * p["samples"] < bench.L2_FLUSH_BYTES
            R = max(1, -(-bench.L2_FLUSH_BYTES // (16 * p["samples"])))
            assert 16 * p["samples"] * R > l2, name
            assert pooled == (name == "dpd1") == (R > 1), name
        else:
            assert p["w"] * p["h"] * p["fmt"] * p["frames"] > l2, name


def test_oracle_only_in_checkers_and_cpu_baseline():
    """oracle/ is test infrastructure: in bench.py only the CPU-baseline legs
    (cpu_motion, cpu_dpd) import it, and nothing in the package or tools/
    does (the product path and the probes never run the checker)."""
    import ast
    import pathlib
    root = pathlib.Path(__file__).resolve().parent.parent

    def importers(path):
        """Names of the functions (or "<module>") holding an oracle import."""
        found = []

        def visit(node, owner):
            for ch in ast.iter_child_nodes(node):
                if isinstance(ch, (ast.FunctionDef, ast.AsyncFunctionDef)):
                    visit(ch, ch.name)
                    continue
                if isinstance(ch, ast.ImportFrom) and (ch.module or "").split(".")[0] == "oracle":
                    found.append(owner)
                elif isinstance(ch, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in ch.names):
                    found.append(owner)
                visit(ch, owner)

        visit(ast.parse(path.read_text()), "<module>")
        return found

    assert set(importers(root / "bench.py")) <= {"cpu_motion", "cpu_dpd"}, importers(root / "bench.py")
    for path in list((root / "paper_1611_03226_b200").rglob("*.py")) + list((root / "tools").rglob("*.py")):
        assert not importers(path), path
