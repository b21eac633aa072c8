"""Drop-in parity on the B200: the reference's own operators (compiled from
its sources) vs include/pdb_patchdb.hpp on the reference's own types --
identical sim_join_pairs sequences (all build sides, probe counts, errors),
apply_transformer histograms and generate+transform features."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_parity")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_parity not built")
def test_reference_operators_vs_b200_adapter():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert r.stdout.startswith("DROPIN OK")
    assert int(r.stdout.split()[2]) > 1000
