"""The band plan (exact tile pruning on two principal projections, join.cu
k_pca_* / k_band_*): the pair set must be identical to the dense screen's
and to the brute-force oracle's, for self and cross joins, every padding
class, shards, degenerate data and non-finite rows.  PDB_JOIN_BAND=1 forces
the plan below its default size threshold; PDB_JOIN_DENSE (dense=True)
disables it."""

import numpy as np
import pytest

from oracle import oracle
from paper_1812_07607_b200 import patchdb, workloads

pytestmark = pytest.mark.gpu


def _pairs(res):
    return set(zip(res.left.tolist(), res.right.tolist()))


def _check_vs_oracle(L, R, tau, self_join):
    got = patchdb.sim_join(L, R, tau, self_join=self_join)
    ol, orr, od = oracle.sim_join(L, R, tau, self_join=self_join)
    assert np.array_equal(got.left, ol) and np.array_equal(got.right, orr)
    assert np.array_equal(got.dist, od.astype(np.float32))
    return got


@pytest.fixture
def forced(monkeypatch):
    monkeypatch.setenv("PDB_JOIN_BAND", "1")


@pytest.mark.parametrize("d", [1, 3, 17, 64, 100, 128])
def test_forced_band_self_matches_oracle(forced, d):
    x = workloads.clusters(5000 + 37 * d, d, 60, 0.02, True, d)
    _check_vs_oracle(x, None, 0.05 if d > 3 else 0.002, True)


@pytest.mark.parametrize("n,m,d,tau", [(3000, 4100, 64, 0.3), (777, 2000, 128, 0.6),
                                       (2048, 257, 5, 0.05), (1, 5000, 64, 2.0)])
def test_forced_band_cross_matches_oracle(forced, n, m, d, tau):
    rng = np.random.default_rng(n + m)
    L = rng.random((n, d), dtype=np.float32)
    R = np.concatenate([L[: min(n, m) // 2] + 1e-3 * rng.standard_normal((min(n, m) // 2, d),
                                                                         dtype=np.float32),
                        rng.random((m - min(n, m) // 2, d), dtype=np.float32)])
    _check_vs_oracle(L, R, tau, False)


def test_forced_band_degenerate_data(forced):
    # identical rows (zero covariance), a single distinct direction, tau = 0
    x = np.zeros((3000, 64), np.float32)
    _check_vs_oracle(x, None, 0.0, True)
    x[::3, 5] = 1.0
    _check_vs_oracle(x, None, 0.0, True)
    _check_vs_oracle(x, None, 0.999, True)
    # everything within tau: no tile may be pruned
    y = workloads.uniform(2500, 64, 4)
    got = _check_vs_oracle(y, None, 100.0, True)
    assert len(got) == 2500 * 2499 // 2


@pytest.mark.parametrize("f16", ["1", "2"])
def test_forced_band_nonfinite_and_huge_rows(forced, monkeypatch, f16):
    # f16 = "2": the same on fp16 copies (NaN / inf rows excluded, 3e30 rows
    # beyond the scale's range forced candidates)
    monkeypatch.setenv("PDB_SCREEN_FP16", f16)
    rng = np.random.default_rng(7)
    x = rng.random((4000, 64), dtype=np.float32)
    x[10] = np.nan
    x[11, 3] = np.inf
    x[12] = -np.inf
    x[13] = 3e30            # beyond the screen's range: always a candidate
    x[14] = 3e30
    x[15] = x[13]
    x[16:40] = x[100:124] + 1e-4
    got = _check_vs_oracle(x, None, 0.05, True)
    assert (13, 15) in _pairs(got) and (13, 14) in _pairs(got)


def test_forced_band_shards_partition(forced):
    x = workloads.clusters(9000, 64, 80, 0.02, True, 11)
    full = patchdb.sim_join(x, None, 0.05, self_join=True)
    parts = [patchdb.sim_join(x, None, 0.05, self_join=True, shard=(k, 3)) for k in range(3)]
    sets = [_pairs(p) for p in parts]
    assert sum(len(s) for s in sets) == len(full)
    assert set().union(*sets) == _pairs(full)


def _band_vs_dense(L, R, tau, self_join):
    import torch
    Lt = torch.from_numpy(L).cuda()
    Rt = None if R is None else torch.from_numpy(R).cuda()
    b = patchdb.sim_join_device(Lt, Rt, tau, self_join=self_join, sort=True)
    bl, br, bd = (t.cpu().numpy() for t in b.to_torch(Lt.device))
    tiles_b = b.stats.tiles
    dn = patchdb.sim_join_device(Lt, Rt, tau, self_join=self_join, sort=True, dense=True)
    dl, dr, dd = (t.cpu().numpy() for t in dn.to_torch(Lt.device))
    assert np.array_equal(bl, dl) and np.array_equal(br, dr) and np.array_equal(bd, dd)
    return tiles_b, dn.stats.tiles, len(bl)


def test_default_band_config2_features():
    fr, _ = workloads.frames(600, 480, 640, seed=2)
    h = patchdb.featurize_tiles(fr, 60, 80, 4, "joint")
    tb, td, n = _band_vs_dense(h, None, 0.05, True)
    assert n > 0 and tb < 0.7 * td
    # sampled rows against the brute-force oracle
    res = patchdb.sim_join(h, None, 0.05, self_join=True)
    for r0 in (0, 20_000, 38_300):
        ol, orr, od = oracle.sim_join(h, None, 0.05, self_join=True, rows=(r0, r0 + 100))
        m = (res.left >= r0) & (res.left < r0 + 100)
        assert np.array_equal(res.left[m], ol) and np.array_equal(res.right[m], orr)


def test_default_band_cross_d128_planted():
    """Config-3 distribution at 65,536 rows: band == dense, both == the exact
    CPU join, and every planted pair present."""
    L, R, pl, pr = workloads.config3(n=65_536)
    tb, td, n = _band_vs_dense(L, R, 0.02, False)
    assert n > 0 and tb < 0.5 * td
    res = patchdb.sim_join(L, R, 0.02)
    ol, orr, od = oracle.sim_join_pruned(L, R, 0.02)
    assert np.array_equal(res.left, ol) and np.array_equal(res.right, orr)
    got = set(zip(res.left.tolist(), res.right.tolist()))
    assert all((a, b) in got for a, b in zip(pl.tolist(), pr.tolist()))


def test_default_band_skewed_self():
    x = workloads.config5(131_072)
    tb, td, n = _band_vs_dense(x, None, 0.01, True)
    assert n > 100_000 and tb < td


def test_forced_band_tf32_copies(forced):
    x = workloads.clusters(6000, 64, 70, 0.02, True, 5)
    got = patchdb.sim_join(x, None, 0.05, self_join=True, tf32=True)
    ol, orr, od = oracle.sim_join(x, None, 0.05, self_join=True)
    assert np.array_equal(got.left, ol) and np.array_equal(got.right, orr)


def test_band_rule_small_joins(monkeypatch):
    """Single-GPU self-joins take the band plan from 4,096 dense tiles
    (config 1's 20,000 rows: 6,319), smaller ones (12,000 rows: 2,303
    tiles) stay dense; both give the oracle's pairs."""
    import torch
    for n, band in ((12_000, False), (20_000, True)):
        xh = workloads.config1(n, seed=1)
        x = torch.from_numpy(xh).cuda()
        monkeypatch.delenv("PDB_JOIN_BAND", raising=False)
        r = patchdb.sim_join_device(x, None, 0.05, self_join=True, sort=True)
        monkeypatch.setenv("PDB_JOIN_BAND", "0")
        d = patchdb.sim_join_device(x, None, 0.05, self_join=True, sort=True)
        nb = -(-n // 128)
        assert d.stats.tiles == sum(-(-n // 256) - rb // 2 for rb in range(nb))
        assert (r.stats.launches > d.stats.launches) == band, n
        got = [t.cpu().numpy() for t in r.to_torch(x.device)]
        want = [t.cpu().numpy() for t in d.to_torch(x.device)]
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
        if n == 12_000:
            ol, orr, od = oracle.sim_join(xh, None, 0.05, self_join=True, threads=8)
            assert np.array_equal(got[0], ol) and np.array_equal(got[1], orr)
            assert np.array_equal(got[2], od.astype(np.float32))


def test_sharded_band_plan_deterministic_order(forced):
    """Sharded self-joins need every rank to build the same row order: the
    stable counting sort (k_rank_*) gives the shards an exact partition of the
    pair set on clustered data with heavily shared sort keys, and identical
    shard outputs on repeated calls."""
    x = workloads.config5(60_000)
    full = _pairs(patchdb.sim_join(x, None, 0.01, self_join=True))
    for P in (2, 5):
        parts = [patchdb.sim_join(x, None, 0.01, self_join=True, shard=(k, P)) for k in range(P)]
        sets = [_pairs(p) for p in parts]
        assert sum(len(s) for s in sets) == len(full)
        assert set().union(*sets) == full
    a = patchdb.sim_join(x, None, 0.01, self_join=True, shard=(1, 3))
    b = patchdb.sim_join(x, None, 0.01, self_join=True, shard=(1, 3))
    assert np.array_equal(a.left, b.left) and np.array_equal(a.right, b.right)


def _device_join(x, R, tau, self_join):
    import torch
    xt = torch.from_numpy(x).cuda()
    rt = None if R is None else torch.from_numpy(R).cuda()
    r = patchdb.sim_join_device(xt, rt, tau, self_join=self_join, sort=True)
    out = [t.cpu().numpy() for t in r.to_torch(xt.device)]
    return out, r.stats.candidates


@pytest.mark.parametrize("case", ["config5", "config3", "forced_d17"])
def test_fp16_copies_same_pairs_fewer_candidates(monkeypatch, case):
    """Band-plan joins can screen fp16 copies of the scaled centred rows
    (fp16_scale; forced here with PDB_SCREEN_FP16=2): the same pairs and
    distances as the bf16 copies (PDB_SCREEN_FP16=0) and the oracle, with a
    narrower candidate band."""
    if case == "config5":
        L, R, tau, self_join = workloads.config5(131_072), None, 0.01, True
    elif case == "config3":
        L, R, _, _ = workloads.config3(n=65_536)
        tau, self_join = 0.02, False
    else:
        monkeypatch.setenv("PDB_JOIN_BAND", "1")
        L = workloads.clusters(9000, 17, 80, 0.02, True, 17) * np.float32(300.0) - np.float32(7.0)
        R, tau, self_join = None, 0.05 * 300.0, True
    outs, cands = [], []
    for f16 in ("2", "0"):  # forced fp16 copies, bf16 copies
        monkeypatch.setenv("PDB_SCREEN_FP16", f16)
        o, c = _device_join(L, R, tau, self_join)
        outs.append(o)
        cands.append(c)
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert len(outs[0][0]) > 100
    assert cands[0] <= cands[1]
    if case == "config5":
        assert cands[0] < 0.7 * cands[1]  # the band around tau narrows
    rows = np.arange(0, L.shape[0], 131)
    ol, orr, od = oracle.sim_join_rows(L, R, tau, rows, self_join=self_join)
    m = np.isin(outs[0][0], rows)
    assert np.array_equal(outs[0][0][m], ol) and np.array_equal(outs[0][1][m], orr)
    assert np.array_equal(outs[0][2][m], od.astype(np.float32))


def test_fp16_copies_fall_back_for_wide_ranges(monkeypatch):
    """One row 1e15 away sets the fp16 scale so low that the other rows
    would land in fp16's subnormals; the join keeps bf16 copies (same
    candidates as PDB_SCREEN_FP16=0) and stays exact."""
    monkeypatch.setenv("PDB_JOIN_BAND", "1")
    x = workloads.clusters(6000, 64, 70, 0.02, True, 5)
    x[17] = 1e15
    cands = []
    for f16 in ("2", "0"):
        monkeypatch.setenv("PDB_SCREEN_FP16", f16)
        got = patchdb.sim_join(x, None, 0.05, self_join=True)
        cands.append(got)
    ol, orr, od = oracle.sim_join(x, None, 0.05, self_join=True)
    for got in cands:
        assert np.array_equal(got.left, ol) and np.array_equal(got.right, orr)
        assert np.array_equal(got.dist, od.astype(np.float32))
    _, c1 = _device_join(x, None, 0.05, True)
    monkeypatch.setenv("PDB_SCREEN_FP16", "2")
    _, c2 = _device_join(x, None, 0.05, True)
    assert c1 == c2


def test_fp16_copies_chosen_for_candidate_heavy_joins(monkeypatch):
    """By default a band-plan join re-makes its copies in fp16 when the
    sampled screen shows >= 4 candidates per column row (config 5's
    distribution at 1M rows): identical output to bf16 copies throughout,
    far fewer candidates, exact on sampled rows."""
    x = workloads.config5(1 << 20)
    outs, cands = [], []
    for f16 in ("1", "0"):
        monkeypatch.setenv("PDB_SCREEN_FP16", f16)
        o, c = _device_join(x, None, 0.01, True)
        outs.append(o)
        cands.append(c)
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert len(outs[0][0]) > 10_000_000
    assert cands[0] < 0.6 * cands[1]
    rows = np.arange(0, x.shape[0], 16_411)
    ol, orr, od = oracle.sim_join_rows(x, None, 0.01, rows, self_join=True)
    m = np.isin(outs[0][0], rows)
    assert np.array_equal(outs[0][0][m], ol) and np.array_equal(outs[0][1][m], orr)
    assert np.array_equal(outs[0][2][m], od.astype(np.float32))
