"""Plan-file JSON surface: run_query / run_etl against the
reference's own run_query on the same plan files and store fixtures
(tests/golden/plans_golden.json.gz, minted by make_golden.py plans from
oracle/_ref).  Tuples are compared with ids, shapes, metadata, lineage
(op, source, region, params digest) and data; the materialized ETL
collection files must be byte-identical to PatchCollection::materialize's.

Histogram ETLs run K1 and joins run K2/K3, so those cases are GPU tests;
pixel-only ETLs, plan parsing, validation and metadata operators run here."""

import gzip
import hashlib
import json
import os

import pytest

from paper_1812_07607_b200 import patchdb, plans

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SDIR = os.path.join(GOLD, "stores")


def _gold():
    with gzip.open(os.path.join(GOLD, "plans_golden.json.gz"), "rt") as f:
        return json.load(f)


G = _gold()


def _doc(doc, tmp):
    return doc.replace("@STORES@", SDIR).replace("@OUT@", str(tmp))


def _norm(x):
    return json.loads(json.dumps(x))


def _check_case(case, tmp):
    patchdb.reset_patch_ids(1)
    doc = _doc(case["doc"], tmp)
    if "error" in case:
        with pytest.raises(RuntimeError) as ei:
            plans.run_query(doc, with_data=case["with_data"], with_lineage=True)
        assert not isinstance(ei.value, patchdb.DeviceError), ei.value
        assert str(ei.value) == case["error"]
        return
    r = plans.run_query(doc, with_data=case["with_data"], with_lineage=True)
    got = _norm(r["tuples"])
    want = case["tuples"]
    assert len(got) == len(want)
    for k, (a, b) in enumerate(zip(got, want)):
        assert a == b, (k, a, b)
    sha = hashlib.sha256(open(os.path.join(tmp, f"etl_{case['etl']}.pdbc"), "rb").read())
    assert sha.hexdigest() == G["etl_sha"][case["etl"]]
    assert r["records_read"] >= 0 and r["frames_decoded"] == 0
    assert r["stats_csv"].startswith("op,ms,tuples_out,index_probes\n")


CPU_CASES = [c for c in G["cases"] if not c["gpu"]]
GPU_CASES = [c for c in G["cases"] if c["gpu"]]


@pytest.mark.parametrize("case", CPU_CASES, ids=[c["name"] for c in CPU_CASES])
def test_pixel_plans_match_reference(case, tmp_path):
    _check_case(case, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=[c["name"] for c in GPU_CASES])
def test_histogram_plans_match_reference(case, tmp_path):
    _check_case(case, tmp_path)


def _error_cases(tmp, allow_device):
    n_dev = 0
    for e in G["errors"]:
        doc = _doc(e["doc"], tmp)
        patchdb.reset_patch_ids(1)
        with pytest.raises(RuntimeError) as ei:
            plans.run_query(doc)
        if isinstance(ei.value, patchdb.DeviceError) and allow_device:
            n_dev += 1
            continue
        msg = str(ei.value).replace(SDIR, "@STORES@").replace(str(tmp), "@OUT@")
        if "parse_error" in (e["error"] or ""):
            # nlohmann's and Python's JSON parser word syntax errors differently
            assert isinstance(ei.value, patchdb.ValidationError)
            assert msg.startswith("plan file: ")
        else:
            assert msg == e["error"], (e["doc"], msg)
    return n_dev


def test_plan_errors_match_reference(tmp_path):
    # without a GPU only the case that reaches K1 (an unregistered collection
    # is found after the histogram ETL ran) stops at DeviceError
    assert _error_cases(tmp_path, allow_device=True) <= 1


@pytest.mark.gpu
def test_plan_errors_match_reference_gpu(tmp_path):
    assert _error_cases(tmp_path, allow_device=False) == 0


def test_run_etl_pixels_byte_identical(tmp_path):
    case = next(c for c in CPU_CASES if c["name"] == "scan_P")
    doc = json.loads(_doc(case["doc"], tmp_path))
    del doc["plan"]
    patchdb.reset_patch_ids(1)
    r = plans.run_etl(json.dumps(doc))
    assert r == {"patches": 128, "output": doc["etl"]["output"], "indexes": []}
    sha = hashlib.sha256(open(doc["etl"]["output"], "rb").read()).hexdigest()
    assert sha == G["etl_sha"]["P"]
    # reopened through the collection reader: same patches, same bytes back
    pats = plans.PatchCollection.open(doc["etl"]["output"]).patches
    assert [p.patch_id for p in pats] == [t[0]["id"] for t in case["tuples"]]
    again = plans.PatchCollection.materialize(pats, str(tmp_path / "again.pdbc"))
    assert again.patch_count() == 128
    assert open(tmp_path / "again.pdbc", "rb").read() == open(doc["etl"]["output"], "rb").read()
    st = plans.collection_stats(doc["etl"]["output"])
    assert st["patches"] == 128 and st["frames_covered"] == 16 and st["indexes"] == []


def test_reference_collections_roundtrip(tmp_path):
    """Collections the reference materialized (r4, r8) read back and
    re-serialize to the identical file."""
    for name in ("r4", "r8"):
        path = os.path.join(SDIR, f"{name}.pdbc")
        col = plans.PatchCollection.open(path)
        assert col.patch_count() == 96
        out = tmp_path / f"{name}.pdbc"
        plans.PatchCollection.materialize(col.patches, str(out))
        assert open(out, "rb").read() == open(path, "rb").read()
        ps = plans.collection_patches(path, with_data=True)
        assert len(ps) == 96 and len(ps[0]["data"]) == (12 if name == "r4" else 24)
        assert isinstance(ps[0]["meta"]["bbox"], tuple)


def test_store_stats():
    st = plans.store_stats(os.path.join(SDIR, "segmented_lossy4_c8.pdb"))
    assert st["frames"] == 16 and (st["width"], st["height"]) == (48, 32)
    assert st["layout"] == "segmented_file" and st["quality"] == "high"
    assert st["clip_len"] == 8 and st["video_id"] == "v"


def test_unsupported_features_raise(tmp_path):
    base = {"collections": {"r4": os.path.join(SDIR, "r4.pdbc")}}
    for plan in ({"op": "backtrace", "input": {"op": "scan", "collection": "r4"}},
                 {"op": "index_join", "left": {"op": "scan", "collection": "r4"},
                  "collection": "r4", "index": "i", "probe_key": "frameno"}):
        with pytest.raises(plans.UnsupportedError):
            plans.run_query(json.dumps(dict(base, plan=plan)))
    with pytest.raises(plans.UnsupportedError):
        plans.run_query(json.dumps(dict(base, plan={"op": "scan", "collection": "r4"},
                                        load_indexes=[{"collection": "r4", "name": "i"}])))
