"""Small-shape runs of every kernel group, for the checked build
(PDB_CUDA_LIB=paper_1812_07607_b200/libpdb_cuda_checked.so; tests/
test_checked_gpu.py): K1 (TMA-fed joint histogram, per-channel, f32 path),
K2 (1-SM screen, the cta_group::2 pair screen, tf32, the band plan), K3
(row-major and grouped re-checks, cosine), dedup rounds, the sharded plan.
Each case checks its result against the oracle, so a clean run is also a
correct one.  Usage: python tools/sanitize_cases.py [case ...]"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402


def _eq_join(res, L, R, tau, self_join):
    ol, orr, od = oracle.sim_join(L, R, tau, self_join=self_join)
    assert np.array_equal(res.left, ol) and np.array_equal(res.right, orr), "pairs differ"
    assert np.array_equal(res.dist, od.astype(np.float32)), "distances differ"


def k1():
    fr, _ = workloads.frames(3, 480, 640, seed=2)
    for mode, b in (("joint", 4), ("per_channel", 4), ("per_channel", 8)):
        got = patchdb.featurize_tiles(fr, 60, 80, b, mode)
        want = oracle.featurize_tiles(fr, 60, 80, b, 1 if mode == "joint" else 0)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    rng = np.random.default_rng(1)
    odd = rng.integers(0, 256, (2, 37, 53, 3), dtype=np.uint8)
    assert np.array_equal(patchdb.featurize_tiles(odd, 7, 9, 4, "joint"),
                          oracle.featurize_tiles(odd, 7, 9, 4, 1))
    px = rng.integers(0, 256, (5, 12, 16, 3)).astype(np.float32)
    assert np.array_equal(patchdb.color_histogram(px, 8), oracle.color_histogram(px, 8, 0))


def k2_dense():
    x = workloads.config1(3000, seed=1)
    _eq_join(patchdb.sim_join(x, None, 0.05, self_join=True), x, None, 0.05, True)
    rng = np.random.default_rng(2)
    L = rng.random((700, 100), dtype=np.float32)
    R = np.concatenate([L[:300] + 1e-3, rng.random((300, 100), dtype=np.float32)]).astype(np.float32)
    _eq_join(patchdb.sim_join(L, R, 0.5), L, R, 0.5, False)
    _eq_join(patchdb.sim_join(L, R, 0.5, tf32=True), L, R, 0.5, False)
    W = rng.random((300, 300), dtype=np.float32)       # DP > 128: streamed A
    _eq_join(patchdb.sim_join(W, W[::-1].copy(), 6.5), W, W[::-1].copy(), 6.5, False)


def k2_pair():
    os.environ["PDB_SCREEN_PAIR"] = "1"
    try:
        x = workloads.config1(3000, seed=3)
        _eq_join(patchdb.sim_join(x, None, 0.05, self_join=True), x, None, 0.05, True)
    finally:
        del os.environ["PDB_SCREEN_PAIR"]


def band():
    os.environ["PDB_JOIN_BAND"] = "1"
    try:
        x = workloads.config1(4000, seed=4)
        _eq_join(patchdb.sim_join(x, None, 0.05, self_join=True), x, None, 0.05, True)
        L, R, _, _ = workloads.config3(n=6000)
        _eq_join(patchdb.sim_join(L, R, 0.02), L, R, 0.02, False)
        parts = [patchdb.sim_join(x, None, 0.05, self_join=True, shard=(k, 2)) for k in range(2)]
        assert sum(len(p) for p in parts) == len(patchdb.sim_join(x, None, 0.05, self_join=True))
    finally:
        del os.environ["PDB_JOIN_BAND"]


def k3_grouped():
    os.environ["PDB_K3_GROUPED"] = "2"
    try:
        x = workloads.config5(8192)
        _eq_join(patchdb.sim_join(x, None, 0.01, self_join=True), x, None, 0.01, True)
        y = workloads.clusters(3000, 61, 40, 0.02, True, 6)
        _eq_join(patchdb.sim_join(y, None, 0.05, self_join=True), y, None, 0.05, True)
    finally:
        del os.environ["PDB_K3_GROUPED"]


def cosine():
    x = workloads.config4(1500, d=128, seed=3, plant_frac=0.05, plant_sigma=0.15)
    b = workloads.bf16_bits(x)
    res = patchdb.cosine_join_bf16(b, None, 0.95, self_join=True)
    ol, orr, oc = oracle.cosine_join_bf16(b, None, 0.95, self_join=True)
    assert np.array_equal(res.left, ol) and np.array_equal(res.right, orr)


def dedup():
    x = workloads.config1(2500, seed=7)
    g = patchdb.dedup(x, 0.05)
    rep_of, nr = oracle.dedup(x, 0.05)
    assert np.array_equal(g.rep_of, rep_of) and len(g.reps) == nr


def fp16_filter():
    """fp16 screen copies (forced) and the K3 fp32 pre-filter (bf16 copies,
    grouped), against the oracle."""
    for env in ({"PDB_JOIN_BAND": "1", "PDB_SCREEN_FP16": "2"},
                {"PDB_JOIN_BAND": "1", "PDB_SCREEN_FP16": "0", "PDB_K3_GROUPED": "2"}):
        os.environ.update(env)
        try:
            x = workloads.config5(8192)
            _eq_join(patchdb.sim_join(x, None, 0.01, self_join=True), x, None, 0.01, True)
            L, R, _, _ = workloads.config3(n=6000)
            _eq_join(patchdb.sim_join(L, R, 0.02), L, R, 0.02, False)
        finally:
            for k in env:
                del os.environ[k]


def fused():
    """pdb_featurize_join_dev (K1's first-round count, the PCA beside it)."""
    import ctypes as C
    import torch
    from paper_1812_07607_b200 import _capi as capi
    lib = capi.lib()
    fr, _ = workloads.frames(150, 480, 640, seed=7)
    d = torch.from_numpy(fr).cuda()
    feats = torch.empty(150 * 64, 64, device="cuda")
    o = capi.JoinOpts()
    o.flags = capi.PDB_JOIN_SELF
    p = patchdb.DevicePairs()
    assert lib.pdb_featurize_join_dev(d.data_ptr(), 150, 480, 640, 60, 80, 4, 1, 0.05, C.byref(o),
                                      feats.data_ptr(), C.byref(p._p), C.byref(p.stats)) == 0
    torch.cuda.synchronize()
    f = feats.cpu().numpy()
    assert np.array_equal(f.view(np.uint32), oracle.featurize_tiles(fr, 60, 80, 4, 1).view(np.uint32))
    l, r, dd = (t.cpu().numpy() for t in p.to_torch(d.device))
    k = np.lexsort((r, l))
    ol, orr, od = oracle.sim_join(f, None, 0.05, self_join=True)
    assert np.array_equal(l[k], ol) and np.array_equal(r[k], orr)
    assert np.array_equal(dd[k], od.astype(np.float32))


CASES = {"k1": k1, "k2_dense": k2_dense, "k2_pair": k2_pair, "band": band,
         "k3_grouped": k3_grouped, "cosine": cosine, "dedup": dedup,
         "fp16_filter": fp16_filter, "fused": fused}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"case {name} ok", flush=True)
