"""The checked build (libpdb_cuda_checked.so: every PDB_DCHECK device-side
bounds check compiled in -- counter addresses and stage reads in K1, work
units and tile indices in K2, candidate columns and permutations in K3, the
counting-sort scatter, the dedup CSR walk) runs every kernel group on small
shapes, each checked against the oracle.  A violated check traps and fails
the run.  compute-sanitizer is closed on this GPU pool (its runs left GPUs
needing a reset), so this is the memcheck substitute; DESIGN.md section 8."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1812_07607_b200", "libpdb_cuda_checked.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(LIB), reason="checked build missing")]


@pytest.mark.parametrize("case", ["k1", "k2_dense", "k2_pair", "band", "k3_grouped", "cosine",
                                  "dedup", "fp16_filter", "fused"])
def test_checked_build_case(case):
    env = dict(os.environ, PDB_CUDA_LIB=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and f"case {case} ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    assert "PDB_DCHECK failed" not in r.stdout + r.stderr
