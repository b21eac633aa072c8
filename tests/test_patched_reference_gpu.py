"""The drop-in proven on the reference itself: /root/reference/proj built
with INTEGRATION.md section 2 applied (oracle/patchdb_b200.patch, built by
oracle/build_patched.sh into oracle/_ref/patched/), so the reference's own
run_sim_join, run_dedup and apply_transformer(color_histogram) call
libpdb_cuda.so.  On the B200:

* the reference's own python smoke tests (tests/python/test_smoke.py) pass
  against the patched pybind11 module;
* the reference's own acceptance program runs; criterion 2 (20k x 20k 24-d,
  tau 0.1: exactly 400,000 pairs, nested-loop == SimJoin) and criterion 10
  (benchmark determinism, q1 = 40 tuples) pass;
* every GPU plan of tests/golden (histogram ETLs, sim_join, dedup, nl_join)
  gives the same run_query result through the patched module as through the
  unpatched one, built from the same sources with the same flags.

Without a GPU the patched build fails loudly (NoDevice) where the B200 path
runs: there is no CPU fallback."""

import gzip
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATCHED = os.path.join(ROOT, "oracle", "_ref", "patched")
UNPATCHED = os.path.join(ROOT, "oracle", "_ref", "unpatched")
GOLD = os.path.join(ROOT, "tests", "golden")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(os.path.join(PATCHED, "acceptance")),
                                 reason="oracle/_ref/patched not built (oracle/build_patched.sh)")]


def _env(path):
    env = dict(os.environ)
    env["PYTHONPATH"] = path
    return env


def test_reference_smoke_tests_on_patched_module(tmp_path):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "--rootdir", str(tmp_path), os.path.join(PATCHED, "test_smoke.py")],
                       cwd=str(tmp_path), env=_env(PATCHED), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "6 passed" in r.stdout


def test_reference_acceptance_on_patched_build():
    r = subprocess.run([os.path.join(PATCHED, "acceptance")], capture_output=True, text=True,
                       timeout=1200)
    lines = {int(l.split()[2]): l for l in r.stdout.splitlines() if l.startswith(("PASS", "FAIL"))}
    print(r.stdout)
    assert len(lines) == 10, r.stdout + r.stderr
    assert lines[2].startswith("PASS") and "400000 matching pairs" in lines[2], lines[2]
    assert lines[10].startswith("PASS"), lines[10]
    # no criterion may fail by an exception (e.g. a device error)
    assert not any("unexpected exception" in l for l in lines.values()), r.stdout
    # criteria 1, 3-6 and 9 exercise storage, indexes and lineage around the path
    for c in (1, 3, 4, 5, 6, 9):
        assert lines[c].startswith("PASS"), lines[c]


_RUNNER = r"""
import hashlib, json, os, sys
import patchdb
cases = json.load(open(sys.argv[1]))
out_dir = sys.argv[2]
res = []
for c in cases:
    d = os.path.join(out_dir, c["name"])
    os.makedirs(d, exist_ok=True)
    doc = c["doc"].replace("@STORES@", sys.argv[3]).replace("@OUT@", d)
    try:
        r = patchdb.run_query(doc, True)
        ent = {k: r[k] for k in ("tuples", "traced", "records_read", "frames_decoded")}
    except RuntimeError as e:
        ent = {"error": str(e)}
    files = sorted(f for f in os.listdir(d))
    ent["files"] = {f: hashlib.sha256(open(os.path.join(d, f), "rb").read()).hexdigest()
                    for f in files}
    res.append(ent)
print(json.dumps(res))
"""


def test_gpu_plans_patched_equal_unpatched(tmp_path):
    with gzip.open(os.path.join(GOLD, "plans_golden.json.gz"), "rt") as f:
        cases = [c for c in json.load(f)["cases"] if c["gpu"]]
    cf = tmp_path / "cases.json"
    cf.write_text(json.dumps(cases))
    outs = []
    for kind, path in (("patched", PATCHED), ("unpatched", UNPATCHED)):
        od = tmp_path / kind
        od.mkdir()
        r = subprocess.run([sys.executable, "-c", _RUNNER, str(cf), str(od),
                            os.path.join(GOLD, "stores")], env=_env(path), capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert len(outs[0]) == len(cases) >= 15
    n_tuples = 0
    for c, a, b in zip(cases, *outs):
        assert a == b, c["name"]
        n_tuples += len(a.get("tuples", []))
    assert n_tuples > 100
