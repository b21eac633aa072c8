"""bench.py contract on the B200: one JSON line with the driver's keys, and
the multi-rank path (torchrun, 2 ranks; gloo so both ranks may share the one
GPU of this box) finds the same pairs as one rank."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks"}


def _run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_contract_one_gpu():
    d = _run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] in ("hbm", "tensor") and 0 < d["roofline"]["frac"]
    assert d["e2e"]["h2d_bytes_per_step"] == 1000 * 480 * 640 * 3
    assert d["pairs"] > 0
    c3 = d["config3"]   # the north-star join, measured in the same run
    assert c3["pairs"] == 5399 and c3["unit"] == "Gpairs/s" and c3["value"] > 0
    assert c3["roofline"]["bound"] == "tensor" and c3["dense_screen"]["pairs"] == 5399
    assert c3["e2e"]["h2d_bytes_per_step"] == 2 * 1048576 * 128 * 4
    _run.one = d


def test_bench_two_ranks_same_pairs():
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
              "--steps", "2", "--warmup", "3", "--no-config3"], env={"PDB_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2
    one = getattr(_run, "one", None) or _run([sys.executable, "bench.py", "--steps", "3",
                                              "--warmup", "3", "--no-cpu-baseline",
                                              "--no-config3"])
    assert d["pairs"] == one["pairs"]


def test_bench_join_workload_c1_and_two_ranks():
    """--workload c1 (join-only line) and its two-rank sharded variant find
    the same pair count (config 1: 1,001,804 pairs)."""
    one = _run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3"])
    assert KEYS <= set(one)
    assert one["unit"] == "Gpairs/s" and one["pairs"] == 1001804
    assert one["cpu_baseline"]["kind"] == "reference" and one["cpu_baseline"]["value"] > 0
    assert 0 < one["roofline"]["frac"] < 1.5
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                "2", "--master-addr", "127.0.0.1", "--master-port", "29534", "bench.py",
                "--gpus", "2", "--workload", "c1", "--steps", "2", "--warmup", "3"],
               env={"PDB_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and two["pairs"] == one["pairs"]


def test_bench_c3_two_ranks_row_sharded():
    """--workload c3 under torchrun (2 ranks; gloo so both share this GPU):
    L row-sharded, R broadcast; the ranks' pairs add up to config 3's 5399."""
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                "2", "--master-addr", "127.0.0.1", "--master-port", "29535", "bench.py",
                "--gpus", "2", "--workload", "c3", "--steps", "2", "--warmup", "3"],
               env={"PDB_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and two["pairs"] == 5399
    assert two["config"]["nL_per_rank"] == 1048576 // 2
    assert "R broadcast once" in two["config"]["parallelism"]
