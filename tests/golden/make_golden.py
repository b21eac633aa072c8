"""Mints tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libpdb_ref.so,
the unmodified proj/ sources compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin both the C restatement (tests/test_oracle.py, CPU) and the
CUDA path (tests/test_*_gpu.py) to the reference's own outputs.  Inputs are
stored alongside outputs, so nothing needs the reference at test time.
"""

from __future__ import annotations

import hashlib
import os
import sys

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


if __name__ == "__main__":
    assert oracle.ref() is not None, "build oracle/_ref first: make -C oracle ref"
    which = sys.argv[1:] or ["hist", "join", "dedup", "nlj", "stores"]
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
