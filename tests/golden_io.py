"""Loads tests/golden/*.npz (minted from the reference by make_golden.py),
regenerating generator-produced inputs and checking their pinned sha256."""

from __future__ import annotations

import hashlib
import os

import numpy as np

from paper_1812_07607_b200 import workloads

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sha(*arrays) -> bytes:
    return hashlib.sha256(b"".join(a.tobytes() for a in arrays)).digest()


def hist_cases():
    z = np.load(os.path.join(HERE, "hist_golden.npz"))
    names = sorted({k.split("__")[0] for k in z.files if k.endswith("__params")})
    cf = None
    for name in names:
        th, tw, b = (int(v) for v in z[f"{name}__params"])
        if f"{name}__frames" in z.files:
            fr = z[f"{name}__frames"]
        else:
            if cf is None:
                cf, _ = workloads.frames(2, 480, 640, seed=2)
            fr = cf
            assert _sha(fr) == z[f"{name}__sha256"].tobytes(), "frame generator drifted"
        yield name, fr, th, tw, b, z[f"{name}__want"]


def f32_case():
    z = np.load(os.path.join(HERE, "hist_golden.npz"))
    return z["f32_clamp_b8__px"], z["f32_clamp_b8__want"]


def _join_inputs(name):
    if name == "clustered_d24":
        a = workloads.clusters(1200, 24, 60, 0.005, False, 4242)
        return a[:600].copy(), a[600:].copy()
    if name == "config1_3k":
        x = workloads.config1(3000, seed=0)
        return x, x
    if name == "uniform_d128":
        u = workloads.uniform(700, 128, 9)
        return u, u[::-1].copy()
    raise KeyError(name)


def join_cases():
    """Yields (name, L, R, tau, sides{side: (left, right, probes)}, dist)."""
    z = np.load(os.path.join(HERE, "join_golden.npz"))
    names = sorted({k.split("__")[0] for k in z.files if k.endswith("__tau")})
    for name in names:
        if f"{name}__L" in z.files:
            L, R = z[f"{name}__L"], z[f"{name}__R"]
        else:
            L, R = _join_inputs(name)
            assert _sha(L, R) == z[f"{name}__sha256"].tobytes(), "workload generator drifted"
        sides = {}
        for s in (0, 1, 2):
            if f"{name}__side{s}_left" in z.files:
                sides[s] = (z[f"{name}__side{s}_left"], z[f"{name}__side{s}_right"],
                            int(z[f"{name}__side{s}_probes"][0]))
        yield name, L, R, float(z[f"{name}__tau"][0]), sides, z[f"{name}__dist"]


def error_tau_negative() -> int:
    z = np.load(os.path.join(HERE, "join_golden.npz"))
    return int(z["error_tau_negative"][0])


def canonical(left, right):
    """Pair set as a sorted structured view for exact comparison."""
    k = (left.astype(np.int64) << 32) | right.astype(np.int64)
    return np.sort(k)


def _dedup_input(name):
    if name == "config1_4k":
        return workloads.config1(4000, seed=0)
    if name == "config2_20f":
        from oracle import oracle
        cf, _ = workloads.frames(20, 480, 640, seed=2)
        return oracle.featurize_tiles(cf, 60, 80, 4, 1)
    raise KeyError(name)


def dedup_cases():
    """(name, X, tau, rep_of, kept) minted from the reference's PlanNode::dedup
    and dedup_stream (tests/golden/make_golden.py dedup)."""
    z = np.load(os.path.join(HERE, "dedup_golden.npz"))
    names = sorted({k.split("__")[0] for k in z.files})
    for name in names:
        if f"{name}__X" in z.files:
            X = z[f"{name}__X"]
        else:
            X = _dedup_input(name)
            assert _sha(X) == z[f"{name}__sha256"].tobytes(), "generator drifted"
        yield name, X, float(z[f"{name}__tau"][0]), z[f"{name}__rep_of"], z[f"{name}__kept"]


def nlj_cases():
    """(name, L, R, radius, left, right) from PlanNode::nl_join(within)."""
    z = np.load(os.path.join(HERE, "nlj_golden.npz"))
    for name in sorted({k.split("__")[0] for k in z.files if k.startswith("nlj_")}):
        yield (name, z[f"{name}__L"], z[f"{name}__R"], float(z[f"{name}__r"][0]),
               z[f"{name}__left"], z[f"{name}__right"])


def q1_cases():
    """(name, frames, bins, tau, a, b) from the reference's q1 plan."""
    z = np.load(os.path.join(HERE, "nlj_golden.npz"))
    for name in sorted({k.split("__")[0] for k in z.files if k.startswith("q1_")}):
        F, H, W, bins = (int(v) for v in z[f"{name}__params"])
        fr, _ = workloads.frames(F, H, W, seed=2)
        assert _sha(fr) == z[f"{name}__sha256"].tobytes(), "frame generator drifted"
        yield name, fr, bins, float(z[f"{name}__tau"][0]), z[f"{name}__a"], z[f"{name}__b"]
