"""Mints tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libpdb_ref.so,
the unmodified proj/ sources compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin both the C restatement (tests/test_oracle.py, CPU) and the
CUDA path (tests/test_*_gpu.py) to the reference's own outputs.  Inputs are
stored alongside outputs, so nothing needs the reference at test time.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1812_07607_b200 import workloads  # noqa: E402


def textured_frame(w, h, f):
    """tests/oracles.hpp:168-177 pixel formula."""
    y, x, c = np.meshgrid(np.arange(h), np.arange(w), np.arange(3), indexing="ij")
    return ((x * 7 + y * 13 + c * 29 + f * 31) & 0xFF).astype(np.uint8)


def solid_frame(w, h, rgb):
    a = np.empty((h, w, 3), np.uint8)
    a[...] = np.array(rgb, np.uint8)
    return a


def hist_fixtures():
    out = {}
    # test_etl.cpp:226-256 textured 16x12 whole-frame patch, B=8
    fr = textured_frame(16, 12, 0)[None]
    out["textured_b8"] = (fr, 12, 16, 8)
    # test_etl.cpp: solid (255,0,129), B=8 -> bins 7 / 0 / 4
    out["solid_b8"] = (solid_frame(8, 8, (255, 0, 129))[None], 8, 8, 8)
    # SPEC.md:372 all-128 patch, B=8 -> 1.0 at 4, 12, 20
    out["gray128_b8"] = (solid_frame(8, 8, (128, 128, 128))[None], 8, 8, 8)
    # test_etl.cpp:278-300 tiles 8x6 over 4 textured 16x12 frames, B=4
    out["tiles_textured_b4"] = (np.stack([textured_frame(16, 12, f) for f in range(4)]), 6, 8, 4)
    # partial edges dropped (test_etl.cpp:91-115): 14x8 frame, tiles 4x3
    out["tiles_partial_b4"] = (textured_frame(14, 8, 0)[None], 3, 4, 4)
    rng = np.random.default_rng(1234)
    frames = rng.integers(0, 256, size=(3, 48, 64, 3), dtype=np.uint8)
    for b in (2, 3, 4, 5, 8, 16, 21, 64, 300):
        out[f"random_b{b}"] = (frames, 12, 16, b)
    # config-2 shaped frames at full resolution (2 frames) with the 60x80 grid
    cf, _ = workloads.frames(2, 480, 640, seed=2)
    out["config2_b4"] = (cf, 60, 80, 4)
    out["config2_b8"] = (cf, 60, 80, 8)
    res = {}
    for name, (fr, th, tw, b) in out.items():
        if name.startswith("config2"):
            # regenerated at test time by workloads.frames(2, seed=2); pin the bytes
            res[f"{name}__sha256"] = np.frombuffer(hashlib.sha256(fr.tobytes()).digest(), np.uint8)
        else:
            res[f"{name}__frames"] = fr
        res[f"{name}__params"] = np.array([th, tw, b], np.int32)
        res[f"{name}__want"] = oracle.ref_featurize_tiles(fr, th, tw, b)
    # float-patch apply_transformer with values >= 256 (clamped to the top bin)
    px = rng.integers(0, 300, size=(5, 7, 9, 3)).astype(np.float32)
    res["f32_clamp_b8__px"] = px
    res["f32_clamp_b8__want"] = oracle.ref_color_histogram(px, 8)
    np.savez_compressed(os.path.join(HERE, "hist_golden.npz"), **res)
    print("hist fixtures:", len(out) + 1)


def join_case(res, name, L, R, tau, sides=(0, 1, 2), store_inputs=True):
    if store_inputs:
        res[f"{name}__L"] = L
        res[f"{name}__R"] = R
    else:
        h = hashlib.sha256(L.tobytes() + R.tobytes()).digest()
        res[f"{name}__sha256"] = np.frombuffer(h, np.uint8)
    res[f"{name}__tau"] = np.array([tau])
    for side in sides:
        li, ri, probes = oracle.ref_sim_join(L, R, tau, side)
        res[f"{name}__side{side}_left"] = li
        res[f"{name}__side{side}_right"] = ri
        res[f"{name}__side{side}_probes"] = np.array([probes], np.int64)
    li = res[f"{name}__side{sides[0]}_left"]
    ri = res[f"{name}__side{sides[0]}_right"]
    res[f"{name}__dist"] = np.array(
        [oracle.ref_euclidean(L[a], R[b]) for a, b in zip(li, ri)], np.float64)


def join_fixtures():
    res = {}
    rng = np.random.default_rng(77)
    # test_query.cpp:268-300 shape: 60 x 40, d=6, U[0,1), tau=0.45
    join_case(res, "random_d6", rng.random((60, 6), dtype=np.float32),
              rng.random((40, 6), dtype=np.float32), 0.45)
    # acceptance.cpp:140-198 shape (scaled): clustered 24-d, sigma 0.005, tau 0.1
    allp = workloads.clusters(1200, 24, 60, 0.005, False, 4242)
    join_case(res, "clustered_d24", allp[:600].copy(), allp[600:].copy(), 0.1, sides=(0,),
              store_inputs=False)
    # config-1 shaped self-join (3,000 rows), reference semantics: ordered
    # pairs incl. (i,i) and both orientations
    x = workloads.config1(3000, seed=0)
    join_case(res, "config1_3k", x, x, 0.05, sides=(2,), store_inputs=False)
    # uniform 128-d (config-3 dimensionality), sparse matches
    u = workloads.uniform(700, 128, 9)
    join_case(res, "uniform_d128", u, u[::-1].copy(), 1.5, sides=(0,), store_inputs=False)
    # exact-radius boundary: test_index.cpp:330-342 and test_query.cpp:128-151
    pts = np.array([[1, 1]] * 5 + [[2, 1]], np.float32)
    join_case(res, "radius_exact", pts, np.array([[1, 1]], np.float32), 1.0)
    join_case(res, "radius_below", pts, np.array([[1, 1]], np.float32), 0.999)
    tri_a = np.array([[0, 0]], np.float32)
    tri_b = np.array([[3, 4]], np.float32)
    join_case(res, "triangle_5", tri_a, tri_b, 5.0)
    join_case(res, "triangle_499", tri_a, tri_b, 4.99)
    # error behaviour: tau < 0 -> ConfigError(1); mixed dims cannot be
    # expressed as arrays, DimensionMismatch is checked in the object API.
    rc = oracle.ref_sim_join(tri_a, tri_b, -0.5, 0)
    res["error_tau_negative"] = np.array([rc])
    np.savez_compressed(os.path.join(HERE, "join_golden.npz"), **res)
    print("join fixtures written")


def dedup_fixtures():
    """PlanNode::dedup through execute() on the reference (ref_dedup): the
    full membership (rep_of) and the kept set of dedup_stream."""
    res = {}
    cases = {}
    # test_query.cpp:331-368: three tight clusters well over tau apart
    cases["test_query_6pts"] = (np.array([[0, 0], [0.01, 0], [1, 1], [0, 0.02], [1.01, 1], [5, 5]],
                                         np.float32), 0.1)
    # exact-distance ties: 0.5 is tau from both kept reps 0 and 1 -> earliest
    cases["tie_1d"] = (np.array([[0.0], [1.0], [0.5], [0.25], [0.75]], np.float32), 0.5)
    rng = np.random.default_rng(95)
    # test_query.cpp:370-389 shape: 300 uniform 3-d points, tau 0.3
    cases["random_300x3"] = (rng.random((300, 3), dtype=np.float32), 0.3)
    cases["random_2000x8"] = (rng.random((2000, 8), dtype=np.float32), 0.5)
    # clustered, config-1 shaped (L1-normalised 64-d), tau 0.05
    cases["config1_4k"] = (workloads.config1(4000, seed=0), 0.05)
    # config-2 tile histograms of 20 frames (1280 tiles), tau 0.05
    cf, _ = workloads.frames(20, 480, 640, seed=2)
    cases["config2_20f"] = (oracle.featurize_tiles(cf, 60, 80, 4, 1), 0.05)
    generated = {"config1_4k", "config2_20f"}  # regenerated at test time, sha-pinned
    for name, (X, tau) in cases.items():
        rep_of, nr = oracle.ref_dedup(X, tau)
        kept = oracle.ref_dedup_stream(X, tau)
        if name in generated:
            res[f"{name}__sha256"] = np.frombuffer(hashlib.sha256(X.tobytes()).digest(), np.uint8)
        else:
            res[f"{name}__X"] = X
        res[f"{name}__tau"] = np.array([tau])
        res[f"{name}__rep_of"] = rep_of
        res[f"{name}__kept"] = kept
        print(name, X.shape, "reps", nr)
    np.savez_compressed(os.path.join(HERE, "dedup_golden.npz"), **res)


def nlj_fixtures():
    """PlanNode::nl_join with a within predicate and the q1 plan, on the
    reference (ref_nl_within, ref_q1)."""
    res = {}
    rng = np.random.default_rng(142)
    cases = {
        "random_50x3_r03": (rng.random((50, 3), dtype=np.float32), rng.random((40, 3), dtype=np.float32), 0.3),
        # test_query.cpp:128-151 shape: 3-4-5 triangle at exactly the radius
        "triangle_r5": (np.array([[0, 0], [3, 4], [6, 8]], np.float32),
                        np.array([[0, 0], [3, 4]], np.float32), 5.0),
        "clustered_d24": (workloads.clusters(300, 24, 20, 0.01, False, 77)[:150].copy(),
                          workloads.clusters(300, 24, 20, 0.01, False, 77)[150:].copy(), 0.05),
    }
    for name, (L, R, r) in cases.items():
        a, b = oracle.ref_nl_within(L, R, r)
        res[f"nlj_{name}__L"] = L
        res[f"nlj_{name}__R"] = R
        res[f"nlj_{name}__r"] = np.array([r])
        res[f"nlj_{name}__left"] = a
        res[f"nlj_{name}__right"] = b
        print(name, len(a))
    for name, (F, H, W, bins, tau) in {"q1_60x96x128_b8": (60, 96, 128, 8, 0.2),
                                       "q1_80x480x640_b4": (80, 480, 640, 4, 0.05)}.items():
        fr, _ = workloads.frames(F, H, W, seed=2)
        a, b = oracle.ref_q1(fr, bins, tau)
        res[f"{name}__params"] = np.array([F, H, W, bins])
        res[f"{name}__tau"] = np.array([tau])
        res[f"{name}__sha256"] = np.frombuffer(hashlib.sha256(fr.tobytes()).digest(), np.uint8)
        res[f"{name}__a"] = a
        res[f"{name}__b"] = b
        print(name, len(a))
    np.savez_compressed(os.path.join(HERE, "nlj_golden.npz"), **res)


def store_fixtures():
    """VideoStore files written by the reference (VideoStore::ingest) for
    every layout, lossless and lossy, and the frames its own scan decodes."""
    sdir = os.path.join(HERE, "stores")
    os.makedirs(sdir, exist_ok=True)
    fr, _ = workloads.frames(16, 32, 48, seed=7, block=8, noise=2, period=6)
    res = {}
    for name, layout, q, cl in [("frame_file", 0, 0, 64), ("encoded_lossless", 1, 0, 64),
                                ("encoded_lossy16", 1, 16, 64), ("segmented_lossless_c5", 2, 0, 5),
                                ("segmented_lossy4_c8", 2, 4, 8)]:
        path = os.path.join(sdir, f"{name}.pdb")
        assert oracle.ref_store_write(fr, path, layout, q, cl) == 0
        full = oracle.ref_store_scan(path, 16, 32, 48)
        part = oracle.ref_store_scan(path, 16, 32, 48, 3, 13)
        res[f"{name}__full_sha"] = np.frombuffer(hashlib.sha256(full.tobytes()).digest(), np.uint8)
        res[f"{name}__part_sha"] = np.frombuffer(hashlib.sha256(part.tobytes()).digest(), np.uint8)
        res[f"{name}__lossless"] = np.array([int(np.array_equal(full, fr))])
        print(name, os.path.getsize(path))
    np.savez_compressed(os.path.join(sdir, "stores_golden.npz"), **res)


# ---- plan files (run_query / run_etl, bindings/py_module.cpp:139-213) -------

def _tiles(bins=None, w=16, h=16, depth=False):
    t = [{"kind": "depth_proxy"}] if depth else []
    if bins:
        t.append({"kind": "color_histogram", "bins": bins})
    return {"kind": "tiles", "tile_w": w, "tile_h": h}, t


def _cmp(op, lhs, rhs, offset=None):
    d = {"kind": "cmp", "op": op, "lhs": lhs, "rhs": rhs}
    if offset is not None:
        d["offset"] = offset
    return d


def _within(a, b, r):
    return {"kind": "within", "slot_a": a, "slot_b": b, "radius": r}


def _fno(slot):
    return {"slot": slot, "key": "frameno"}


PLAN_ETLS = {
    # name: (store fixture, generator, transformers)
    "A": ("segmented_lossless_c5", *_tiles(4)),
    "B": ("encoded_lossy16", {"kind": "whole_image"}, [{"kind": "color_histogram", "bins": 8}]),
    "C": ("frame_file", *_tiles(4, depth=True)),
    "P": ("segmented_lossy4_c8", *_tiles(None, 20, 7, depth=True)),
}
PLAN_COLLECTIONS = {
    # reference-materialized collections the plans open by alias
    "r4": ("encoded_lossless", *_tiles(4)),
    "r8": ("frame_file", *_tiles(8)),
}


def plan_cases():
    """(name, etl key, plan, with_data, gpu) -- every case's expected tuples
    (ids, shape, meta, lineage, data) or error message come from the
    reference's run_query."""
    S = {"op": "scan", "collection": "etl"}
    R4 = {"op": "scan", "collection": "r4"}
    R8 = {"op": "scan", "collection": "r8"}
    dd = lambda x, t: {"op": "dedup", "input": x, "tau": t}
    sj = lambda l, r, t, side=None: dict({"op": "sim_join", "left": l, "right": r, "tau": t},
                                         **({"build_side": side} if side else {}))
    nl = lambda l, r, on: {"op": "nl_join", "left": l, "right": r, "on": on}
    sel = lambda x, p: {"op": "select", "input": x, "pred": p}
    return [
        ("scan_A", "A", S, True, True),
        ("simjoin_self_A", "A", sj(S, S, 0.05), False, True),
        ("simjoin_A_r4_right", "A", sj(S, R4, 0.1, "right"), False, True),
        ("simjoin_A_r4_left", "A", sj(S, R4, 0.1, "left"), False, True),
        ("q1_select_A", "A", sel(sj(S, S, 0.1), _cmp("ne", _fno(0), _fno(1))), False, True),
        ("dedup_A", "A", dd(S, 0.05), True, True),
        ("dedup_A_tau0", "A", dd(S, 0.0), False, True),
        ("dedup_A_neg", "A", dd(S, -1.0), False, True),
        ("nlj_within_A_r4", "A", nl(S, R4, _within(0, 1, 0.1)), False, True),
        ("nlj_and_A_r4", "A", nl(S, R4, {"kind": "and", "parts": [
            _within(1, 0, 0.1), _cmp("ne", _fno(0), _fno(1))]}), False, True),
        ("nlj_or_A_r4", "A", nl(sel(S, _cmp("lt", _fno(0), {"lit": 6})), R4, {"kind": "or", "parts": [
            _within(0, 1, 0.05), _cmp("eq", {"slot": 1, "key": "bbox.x1"}, {"lit": 32})]}),
         False, True),
        ("select_within_pairs", "A", sel(sj(S, R4, 0.2), _within(0, 1, 0.1)), False, True),
        ("countby_dedup_A", "A", {"op": "count_by", "input": dd(S, 0.1), "key": "frameno"},
         False, True),
        ("simjoin_dim_mismatch", "A", sj(S, R8, 0.1), False, True),
        ("nlj_dim_mismatch", "A", nl(S, R8, _within(0, 1, 0.1)), False, True),
        ("dedup_B", "B", dd(S, 0.02), True, True),
        ("simjoin_B", "B", sj(S, S, 0.05), False, True),
        ("scan_C", "C", S, True, True),
        ("simjoin_dedups", "A", sj(dd(S, 0.05), dd(R4, 0.05), 0.1), False, True),
        ("nlj_dedups", "A", nl(dd(S, 0.05), dd(R4, 0.05), _within(0, 1, 0.1)), False, True),
        ("scan_P", "P", S, True, False),
        ("countby_P", "P", {"op": "count_by", "input": S, "key": "depth"}, False, False),
        ("select_P", "P", sel(S, {"kind": "and", "parts": [
            _cmp("ge", {"slot": 0, "key": "bbox.y1"}, {"lit": 14}),
            {"kind": "not", "part": _cmp("eq", _fno(0), {"lit": 3}, 1)}]}), False, False),
        ("nlj_cmp_P", "P", nl(sel(S, _cmp("lt", _fno(0), {"lit": 2})), R4,
                              _cmp("eq", _fno(0), _fno(1), 1)), False, False),
        ("select_box_order_P", "P", sel(S, _cmp("lt", {"slot": 0, "key": "bbox"},
                                                {"lit": [0, 0, 1, 1]})), False, False),
        ("select_slot_P", "P", sel(S, _cmp("eq", {"slot": 2, "key": "frameno"}, {"lit": 1})),
         False, False),
    ]


def plan_error_docs():
    """Malformed plan files: the reference's ValidationError / ConfigError
    messages ("@STORES@" / "@OUT@" are substituted at test time)."""
    etl = {"name": "etl", "store": "@STORES@/frame_file.pdb",
           "generator": {"kind": "tiles", "tile_w": 16, "tile_h": 16},
           "transformers": [{"kind": "color_histogram", "bins": 4}], "output": "@OUT@/e.pdbc"}
    S = {"op": "scan", "collection": "etl"}
    bad = [
        {"etl": etl, "plan": S, "extra": 1},
        {"etl": etl},
        {"etl": etl, "plan": {"op": "frobnicate"}},
        {"etl": etl, "plan": {"op": "sim_join", "left": S, "right": S}},
        {"etl": etl, "plan": {"op": "sim_join", "left": S, "right": S, "tau": "x"}},
        {"etl": etl, "plan": {"op": "sim_join", "left": S, "right": S, "tau": 1, "build_side": "up"}},
        {"etl": etl, "plan": {"op": "select", "input": S, "pred": {"kind": "near"}}},
        {"etl": etl, "plan": {"op": "select", "input": S, "pred": _cmp("approx", _fno(0), _fno(0))}},
        {"etl": etl, "plan": {"op": "select", "input": S, "pred": _cmp("eq", {"slot": -1, "key": "a"},
                                                                         {"lit": 1})}},
        {"etl": etl, "plan": {"op": "select", "input": S, "pred": _cmp("eq", _fno(0), {"lit": {}})}},
        {"etl": etl, "plan": {"op": "dedup", "input": S}},
        {"etl": etl, "plan": {"op": "scan"}},
        {"etl": etl, "plan": {"op": "nl_join", "left": S, "right": S}},
        {"etl": etl, "plan": {"op": "count_by", "input": S}},
        {"etl": dict(etl, generator={"kind": "tiles", "tile_w": 0, "tile_h": 16}), "plan": S},
        {"etl": dict(etl, generator={"kind": "mosaic"}), "plan": S},
        {"etl": dict(etl, transformers=[{"kind": "color_histogram", "bins": 1}]), "plan": S},
        {"etl": dict(etl, transformers=[{"kind": "color_histogram", "bins": 4},
                                        {"kind": "color_histogram", "bins": 4}]), "plan": S},
        {"etl": dict(etl, transformers=[{"kind": "color_histogram", "bins": 4},
                                        {"kind": "depth_proxy"}]), "plan": S},
        {"etl": dict(etl, transformers=[{"kind": "sharpen"}]), "plan": S},
        {"etl": dict(etl, transformers={"kind": "depth_proxy"}), "plan": S},
        {"etl": {k: v for k, v in etl.items() if k != "output"}, "plan": S},
        {"etl": dict(etl, store="@STORES@/missing.pdb"), "plan": S},
        {"etl": etl, "plan": {"op": "scan", "collection": "nope"}},
        {"etl": etl, "plan": {"op": "select", "input": S, "pred": {"kind": "and", "parts": 3}}},
        {"etl": etl, "stores": {"v": 3}, "plan": S},
    ]
    return [json.dumps(d) for d in bad] + ["{not json", "[]"]


def _sub(doc: str, stores: str, out: str) -> str:
    return doc.replace("@STORES@", stores).replace("@OUT@", out)


def plan_doc(etl_key, plan, stores, out):
    store, gen, trans = PLAN_ETLS[etl_key]
    return json.dumps({"etl": {"name": "etl", "store": f"{stores}/{store}.pdb", "generator": gen,
                               "transformers": trans, "output": f"{out}/etl_{etl_key}.pdbc"},
                       "collections": {k: f"{stores}/{k}.pdbc" for k in PLAN_COLLECTIONS},
                       "plan": plan})


def plan_fixtures():
    sdir = os.path.join(HERE, "stores")
    tmp = tempfile.mkdtemp()
    for name, (store, gen, trans) in PLAN_COLLECTIONS.items():
        doc = json.dumps({"etl": {"name": "x", "store": f"{sdir}/{store}.pdb", "generator": gen,
                                  "transformers": trans, "output": f"{sdir}/{name}.pdbc"},
                          "plan": {"op": "scan", "collection": "x"}})
        oracle.ref_run_query(doc, reset_ids=1000)
    res = {"cases": [], "errors": [], "etl_sha": {}}
    for name, key, plan, with_data, gpu in plan_cases():
        doc = plan_doc(key, plan, sdir, tmp)
        try:
            r = oracle.ref_run_query(doc, with_data=with_data, reset_ids=1)
            exp = {"tuples": r["tuples"]}
        except RuntimeError as e:
            exp = {"error": str(e)}
        res["cases"].append({"name": name, "etl": key, "with_data": with_data, "gpu": gpu,
                             "doc": plan_doc(key, plan, "@STORES@", "@OUT@"), **exp})
        res["etl_sha"][key] = hashlib.sha256(open(f"{tmp}/etl_{key}.pdbc", "rb").read()).hexdigest()
        print(name, len(exp.get("tuples", [])), exp.get("error", ""))
    for doc in plan_error_docs():
        try:
            oracle.ref_run_query(_sub(doc, sdir, tmp), reset_ids=1)
            msg = None
        except RuntimeError as e:
            msg = str(e).replace(sdir, "@STORES@").replace(tmp, "@OUT@")
        res["errors"].append({"doc": doc, "error": msg})
        print("error:", msg)
    with gzip.open(os.path.join(HERE, "plans_golden.json.gz"), "wt") as f:
        json.dump(res, f, separators=(",", ":"))


if __name__ == "__main__":
    assert oracle.ref() is not None, "build oracle/_ref first: make -C oracle ref"
    which = sys.argv[1:] or ["hist", "join", "dedup", "nlj", "stores", "plans"]
    if "hist" in which:
        hist_fixtures()
    if "join" in which:
        join_fixtures()
    if "dedup" in which:
        dedup_fixtures()
    if "nlj" in which:
        nlj_fixtures()
    if "stores" in which:
        store_fixtures()
    if "plans" in which:
        plan_fixtures()
