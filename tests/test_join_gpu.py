"""K2 + K3 parity on the B200: the pair set equals the reference's exactly
(golden fixtures from the compiled reference, and the brute-force
restatement at larger sizes); distances within 1e-6 relative of the
reference's fp64 euclidean (fp32 rounding of the exact value)."""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1812_07607_b200 import patchdb, workloads
from tests import golden_io

pytestmark = pytest.mark.gpu

DIST_RTOL = 1e-5   # north_star tolerance; fp32 rounding gives <= 6e-8


def _same_set(gl, gr, wl, wr):
    return np.array_equal(golden_io.canonical(gl, gr), golden_io.canonical(wl, wr))


def _check(res, ol, orr, od):
    assert _same_set(res.left, res.right, ol, orr)
    order = np.lexsort((res.right, res.left))
    assert np.array_equal(res.left[order], ol) and np.array_equal(res.right[order], orr)
    assert np.allclose(res.dist[order].astype(np.float64), od, rtol=DIST_RTOL, atol=0)
    assert np.array_equal(res.dist[order], od.astype(np.float32))


@pytest.mark.parametrize("tf32", [False, True])
def test_golden_cases_cross_join(tf32):
    for name, L, R, tau, sides, dist in golden_io.join_cases():
        li, ri, _ = next(iter(sides.values()))
        res = patchdb.sim_join(L, R, tau, tf32=tf32)
        assert _same_set(res.left, res.right, li, ri), name
        # sorted flag -> ascending (left, right); distances = fp32(euclidean)
        order = np.lexsort((ri, li))
        assert np.array_equal(res.left, li[order]) and np.array_equal(res.right, ri[order]), name
        assert np.array_equal(res.dist, dist[order].astype(np.float32)), name


def test_golden_reference_emission_order_all_build_sides():
    for name, L, R, tau, sides, dist in golden_io.join_cases():
        if L.shape[0] > 1000:
            continue
        lp = [patchdb.Patch(i + 1, L[i], (L.shape[1],)) for i in range(L.shape[0])]
        rp = [patchdb.Patch((1 << 32) + 1 + j, R[j], (R.shape[1],)) for j in range(R.shape[0])]
        for side, (li, ri, probes) in sides.items():
            pr = []
            got = patchdb.sim_join_pairs(lp, rp, tau, patchdb.BuildSide(side), probes=pr)
            gl = np.array([a.patch_id - 1 for a, _ in got], np.int64)
            gr = np.array([b.patch_id - (1 << 32) - 1 for _, b in got], np.int64)
            assert np.array_equal(gl, li) and np.array_equal(gr, ri), (name, side)
            assert pr[0] == probes, (name, side)


def test_golden_config1_selfjoin_reference_semantics():
    for name, L, R, tau, sides, dist in golden_io.join_cases():
        if name != "config1_3k":
            continue
        li, ri, _ = sides[2]
        m = li < ri
        res = patchdb.sim_join(L, None, tau, self_join=True)
        assert _same_set(res.left, res.right, li[m], ri[m])
        full = patchdb.sim_join(L, L, tau)   # ordered, incl. diagonal, like sim_join_pairs(X, X)
        assert _same_set(full.left, full.right, li, ri)


def test_config1_full_selfjoin_vs_oracle():
    x = workloads.config1()
    res = patchdb.sim_join(x, None, 0.05, self_join=True)
    ol, orr, od = oracle.sim_join(x, None, 0.05, self_join=True)
    assert len(ol) > 100_000
    _check(res, ol, orr, od)


@pytest.mark.parametrize("tf32", [False, True])
@pytest.mark.parametrize("d", [1, 2, 3, 5, 12, 24, 31, 32, 33, 63, 64, 65, 96, 100, 128, 129,
                               200, 256, 300, 512, 1000, 2048])
def test_dims_cross_join(d, tf32):
    rng = np.random.default_rng(d)
    L = rng.random((700, d), dtype=np.float32)
    R = np.concatenate([L[rng.integers(0, 700, 300)] +
                        rng.normal(0, 0.01, (300, d)).astype(np.float32),
                        rng.random((500, d), dtype=np.float32)]).astype(np.float32)
    dd = np.sqrt(((L[:, None, :].astype(np.float64) - R[None]) ** 2).sum(-1))
    tau = float(np.quantile(dd, 0.01))
    res = patchdb.sim_join(L, R, tau, tf32=tf32)
    ol, orr, od = oracle.sim_join(L, R, tau, threads=8)
    assert len(ol) > 0
    _check(res, ol, orr, od)


@pytest.mark.parametrize("tf32", [False, True])
@pytest.mark.parametrize("scale", [1e-6, 1e-2, 1.0, 1e3, 1e8])
def test_value_scales_and_offsets(scale, tf32):
    rng = np.random.default_rng(int(scale * 7) % 1000)
    off = rng.normal(0, 50 * scale, (1, 48)).astype(np.float32)
    L = (rng.random((900, 48)) * scale + off).astype(np.float32)
    R = (L[::3] + rng.normal(0, 0.02 * scale, (300, 48))).astype(np.float32)
    tau = 0.2 * scale * np.sqrt(48) * 0.05
    res = patchdb.sim_join(L, R, tau, tf32=tf32)
    ol, orr, od = oracle.sim_join(L, R, tau, threads=8)
    _check(res, ol, orr, od)


@pytest.mark.parametrize("tf32,grouped", [(False, False), (True, False), (False, True)])
def test_boundary_pairs_exactly_at_tau(monkeypatch, tf32, grouped):
    # Pairs whose fp64 distance is EXACTLY tau must be kept (inclusive <=),
    # and tau one ulp below must drop them.  `grouped` forces the re-check
    # through the grouped copy and its fp32 pre-filter (k_recheck_filtered).
    if grouped:
        monkeypatch.setenv("PDB_K3_GROUPED", "2")
    rng = np.random.default_rng(4)
    L = rng.random((513, 24), dtype=np.float32)
    R = L.copy()
    R[:, 0] += np.float32(0.25)          # exact shift: distance exactly 0.25 when representable
    d = np.array([oracle.euclidean(L[i], R[i]) for i in range(len(L))])
    tau = float(np.median(d))
    res = patchdb.sim_join(L, R, tau, tf32=tf32)
    ol, orr, od = oracle.sim_join(L, R, tau, threads=8)
    _check(res, ol, orr, od)
    assert (od == tau).sum() > 0
    below = np.nextafter(tau, 0)
    res2 = patchdb.sim_join(L, R, below, tf32=tf32)
    ol2, orr2, od2 = oracle.sim_join(L, R, below, threads=8)
    _check(res2, ol2, orr2, od2)
    assert len(ol2) < len(ol)


@pytest.mark.parametrize("tf32,grouped", [(False, False), (True, False), (False, True)])
def test_nonfinite_and_huge_rows(monkeypatch, tf32, grouped):
    if grouped:  # huge rows overflow the fp32 pre-filter's sums to +inf
        monkeypatch.setenv("PDB_K3_GROUPED", "2")
    rng = np.random.default_rng(8)
    L = rng.random((300, 16), dtype=np.float32)
    R = L[::-1].copy()
    L[5, 3] = np.nan
    L[6, 0] = np.inf
    R[7, 2] = -np.inf
    L[10] = 3e30    # squares overflow fp32: forced through the exact path
    R[20] = 3e30
    L[11] = 1e19
    R[21] = 1e19
    res = patchdb.sim_join(L, R, 0.3, tf32=tf32)
    ol, orr, od = oracle.sim_join(L, R, 0.3, threads=4)
    _check(res, ol, orr, od)
    assert (5 not in res.left) and (6 not in res.left)


def test_empty_and_tiny_inputs():
    z = np.zeros((0, 8), np.float32)
    one = np.ones((1, 8), np.float32)
    assert len(patchdb.sim_join(z, one, 1.0)) == 0
    assert len(patchdb.sim_join(one, z, 1.0)) == 0
    assert len(patchdb.sim_join(one, None, 1.0, self_join=True)) == 0
    r = patchdb.sim_join(one, one, 0.0)
    assert len(r) == 1 and r.dist[0] == 0.0
    two = np.array([[0, 0], [3, 4]], np.float32)
    r = patchdb.sim_join(two, None, 5.0, self_join=True)
    assert len(r) == 1 and r.dist[0] == 5.0
    assert len(patchdb.sim_join(two, None, 4.99, self_join=True)) == 0


def test_ragged_sizes_tile_edges():
    rng = np.random.default_rng(12)
    for nL, nR in [(1, 257), (127, 1), (129, 255), (257, 513), (1000, 3)]:
        L = rng.random((nL, 20), dtype=np.float32)
        R = rng.random((nR, 20), dtype=np.float32)
        res = patchdb.sim_join(L, R, 0.6)
        ol, orr, od = oracle.sim_join(L, R, 0.6, threads=4)
        _check(res, ol, orr, od)
        s = patchdb.sim_join(L, None, 0.6, self_join=True)
        ol, orr, od = oracle.sim_join(L, None, 0.6, self_join=True, threads=4)
        _check(s, ol, orr, od)


def test_shards_partition_the_pair_set():
    x = workloads.config1(6000, seed=1)
    full = patchdb.sim_join(x, None, 0.05, self_join=True)
    parts = [patchdb.sim_join(x, None, 0.05, self_join=True, shard=(k, 3)) for k in range(3)]
    l = np.concatenate([p.left for p in parts])
    r = np.concatenate([p.right for p in parts])
    assert len(l) == len(full)
    assert _same_set(l, r, full.left, full.right)
    from paper_1812_07607_b200 import shard
    for k, p in enumerate(parts):
        assert np.isin(p.left, shard.shard_rows(k, 3, x.shape[0])).all()


def test_device_entry_and_reuse():
    x = torch.from_numpy(workloads.config1(5000, seed=3)).cuda()
    out = patchdb.DevicePairs()
    a = patchdb.sim_join_device(x, None, 0.05, self_join=True, sort=True, out=out)
    n1 = a.count
    l1, r1, d1 = (t.cpu().numpy() for t in a.to_torch(x.device))
    b = patchdb.sim_join_device(x, None, 0.05, self_join=True, sort=True, out=out)
    assert b.count == n1
    ol, orr, od = oracle.sim_join(x.cpu().numpy(), None, 0.05, self_join=True)
    assert np.array_equal(l1, ol) and np.array_equal(r1, orr)
    assert a.stats.candidates >= a.stats.pairs == n1
    assert a.stats.tiles > 0


def test_featurize_join_pipeline():
    fr, src = workloads.frames(60, 480, 640, seed=2)
    feats, res = patchdb.featurize_join(fr, 60, 80, 4, "joint", 0.05, want_features=True)
    want = oracle.featurize_tiles(fr, 60, 80, 4, 1)
    assert np.array_equal(feats.view(np.uint32), want.view(np.uint32))
    ol, orr, od = oracle.sim_join(want, None, 0.05, self_join=True)
    _check(res, ol, orr, od)


def test_config5_scaled_skewed_output_sampled_rows():
    """Config 5 distribution (20% in 50 tight simplex clusters, tau = 0.01) at
    262,144 rows: dense skewed output.  Rows of a deterministic sample are
    checked exactly against the brute-force oracle; the total is checked
    against the sum of per-row counts on the device."""
    x = workloads.config5(262_144)
    res = patchdb.sim_join(x, None, 0.01, self_join=True, sort=True)
    assert len(res) > 1_000_000
    for r0 in (0, 70_000, 262_000):
        ol, orr, od = oracle.sim_join(x, None, 0.01, self_join=True, rows=(r0, r0 + 64))
        m = (res.left >= r0) & (res.left < r0 + 64)
        assert np.array_equal(res.left[m], ol) and np.array_equal(res.right[m], orr)
        assert np.array_equal(res.dist[m], od.astype(np.float32))


def test_cta_pair_screen_opt_in(monkeypatch):
    """The cta_group::2 screen (PDB_SCREEN_PAIR=1) finds the same pair set as
    the brute-force oracle, self and cross, with ragged edges."""
    monkeypatch.setenv("PDB_SCREEN_PAIR", "1")
    rng = np.random.default_rng(21)
    for n, m, d, tau in [(3000, None, 64, 0.05), (1000, 777, 100, 0.9), (700, None, 17, 0.3)]:
        L = workloads.clusters(n, d, 40, 0.02, True, 3) if m is None else rng.random((n, d), dtype=np.float32)
        R = None if m is None else rng.random((m, d), dtype=np.float32)
        got = patchdb.sim_join(L, R, tau, self_join=m is None)
        ol, orr, od = oracle.sim_join(L, R, tau, self_join=m is None)
        assert np.array_equal(got.left, ol) and np.array_equal(got.right, orr)
        assert np.array_equal(got.dist, od.astype(np.float32))


def test_record_overflow_rescreen(monkeypatch):
    """PDB_TEST_REC_CAP caps the first pass's candidate-record buffer: the
    join must detect the overflow, re-run the screen with the exact record
    count (screen_passes == 2) and still return the oracle's pair set; the
    same on a join large enough for the sampled sizing pass."""
    x = workloads.config1()
    ol, orr, od = oracle.sim_join(x, None, 0.05, self_join=True)
    monkeypatch.setenv("PDB_TEST_REC_CAP", "1000")
    xt = torch.from_numpy(x).cuda()
    r = patchdb.sim_join_device(xt, None, 0.05, self_join=True, sort=True)
    assert r.stats.screen_passes == 2 and r.stats.candidates > 1000
    l_, r_, d_ = (t.cpu().numpy() for t in r.to_torch(xt.device))
    assert np.array_equal(l_, ol) and np.array_equal(r_, orr)
    assert np.array_equal(d_, od.astype(np.float32))
    big = workloads.config5(1 << 20)
    bt = torch.from_numpy(big).cuda()
    monkeypatch.delenv("PDB_TEST_REC_CAP")
    ref = patchdb.sim_join_device(bt, None, 0.01, self_join=True, sort=True)
    want = [t.cpu().numpy() for t in ref.to_torch(bt.device)]
    assert ref.stats.screen_passes == 1
    ref.free()
    monkeypatch.setenv("PDB_TEST_REC_CAP", "4096")
    got = patchdb.sim_join_device(bt, None, 0.01, self_join=True, sort=True)
    assert got.stats.screen_passes == 2
    for a, b in zip(want, (t.cpu().numpy() for t in got.to_torch(bt.device))):
        assert np.array_equal(a, b)
    rows = np.arange(0, big.shape[0], 16_411)
    ol, orr, od = oracle.sim_join_rows(big, None, 0.01, rows, self_join=True)
    m = np.isin(want[0], rows)
    assert np.array_equal(want[0][m], ol) and np.array_equal(want[1][m], orr)


def test_short_heavy_join_rescreens_on_fp16_copies():
    """A band-plan join too short for the sampled sizing pass whose first
    screen overflows the default record buffer with a candidate-heavy output
    (config 5's distribution at 262k rows) re-screens on fp16 copies: two
    passes, far fewer candidates than the bf16 copies give, exact pairs."""
    big = workloads.config5(262_144)
    bt = torch.from_numpy(big).cuda()
    r = patchdb.sim_join_device(bt, None, 0.01, self_join=True, sort=True)
    assert r.stats.screen_passes == 2
    assert r.stats.candidates < 0.7 * 10_900_000  # bf16 copies: ~10.9 M
    got = [t.cpu().numpy() for t in r.to_torch(bt.device)]
    rows = np.arange(0, big.shape[0], 2049)
    ol, orr, od = oracle.sim_join_rows(big, None, 0.01, rows, self_join=True)
    m = np.isin(got[0], rows)
    assert np.array_equal(got[0][m], ol) and np.array_equal(got[1][m], orr)
    assert np.array_equal(got[2][m], od.astype(np.float32))


def test_pair_overflow_rerun(monkeypatch):
    """PDB_TEST_OUT_CAP caps the first pair buffer: only the re-check re-runs."""
    x = workloads.config1(8000, seed=5)
    ol, orr, od = oracle.sim_join(x, None, 0.05, self_join=True)
    monkeypatch.setenv("PDB_TEST_OUT_CAP", "100")
    res = patchdb.sim_join(x, None, 0.05, self_join=True)
    assert len(ol) > 100
    _check(res, ol, orr, od)


@pytest.mark.parametrize("case", ["config5_self", "band_cross_permR", "odd_d61"])
def test_grouped_recheck_bit_identical(monkeypatch, case):
    """The grouped re-check (k_group_copy + k_recheck_filtered, or
    k_recheck<1|2> without the fp32 pre-filter; forced with
    PDB_K3_GROUPED=2) and the row-major one (=0) return bit-identical sorted
    output, equal to the oracle: self join, a band-plan cross join (column
    permutation permR) and d % 8 != 0."""
    rng = np.random.default_rng(61)
    if case == "config5_self":
        L, R, tau, self_join = workloads.config5(131_072), None, 0.01, True
    elif case == "band_cross_permR":
        L, R, _, _ = workloads.config3(n=65_536)
        tau, self_join = 0.02, False
    else:
        L = workloads.clusters(20_000, 61, 150, 0.02, True, 61)
        R = (L[rng.integers(0, 20_000, 9000)] + rng.normal(0, 2e-4, (9000, 61))).astype(np.float32)
        tau, self_join = 0.01, False
    Lt = torch.from_numpy(L).cuda()
    Rt = None if R is None else torch.from_numpy(R).cuda()
    outs = []
    # grouped with the fp32 pre-filter (k_recheck_filtered: bf16 screen
    # copies), grouped without it (PDB_K3_FILTER=0: k_recheck<1|2>),
    # grouped after an fp16 screen (band plans), and row-major
    for mode, filt, f16 in (("2", "1", "0"), ("2", "0", "0"), ("2", "1", "1"), ("0", "1", "1")):
        monkeypatch.setenv("PDB_K3_GROUPED", mode)
        monkeypatch.setenv("PDB_K3_FILTER", filt)
        monkeypatch.setenv("PDB_SCREEN_FP16", f16)
        r = patchdb.sim_join_device(Lt, Rt, tau, self_join=self_join, sort=True)
        outs.append([t.cpu().numpy() for t in r.to_torch(Lt.device)])
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)
    assert len(outs[0][0]) > 300
    rows = np.arange(0, L.shape[0], 97)
    ol, orr, od = oracle.sim_join_rows(L, R, tau, rows, self_join=self_join)
    m = np.isin(outs[0][0], rows)
    assert np.array_equal(outs[0][0][m], ol) and np.array_equal(outs[0][1][m], orr)
    assert np.array_equal(outs[0][2][m], od.astype(np.float32))


def test_nan_tau_matches_nothing_like_the_reference():
    """The reference rejects only tau < 0 (src/query.cpp:488); a NaN tau
    passes and emits no pairs (every `euclidean <= NaN` is false)."""
    x = workloads.config1(3000, seed=2)
    assert len(patchdb.sim_join(x, None, float("nan"), self_join=True)) == 0
    assert len(patchdb.sim_join(x, x, float("nan"))) == 0
    g = patchdb.dedup(x, float("nan"))
    assert len(g.reps) == 3000
    with pytest.raises(patchdb.ConfigError):
        patchdb.sim_join(x, None, -1e-300, self_join=True)


def test_release_caches():
    from paper_1812_07607_b200 import _capi as capi
    x = workloads.config5(262_144)
    a = patchdb.sim_join(x, None, 0.01, self_join=True)
    assert capi.lib().pdb_release_caches() == 0
    b = patchdb.sim_join(x, None, 0.01, self_join=True)
    assert np.array_equal(a.left, b.left) and np.array_equal(a.right, b.right)


@pytest.mark.parametrize("variant", ["band", "dense", "nofold", "tf32", "pair"])
@pytest.mark.parametrize("n,d", [(5000, 1), (9000, 1), (6000, 2), (4000, 8), (3000, 64)])
def test_bf16_rounding_bound(monkeypatch, variant, n, d):
    """Rows on a line far from the screen copies' centre, neighbours 0.9 tau
    apart: the bf16 copy's rounding error reaches its worst case (half an
    ulp = 2^-8 of the rounded value) on every coordinate at once, so a margin
    that underestimates it loses pairs (r01's 2^-9 did)."""
    if variant == "nofold":
        monkeypatch.setenv("PDB_NO_FOLD", "1")
    if variant == "pair":
        monkeypatch.setenv("PDB_SCREEN_PAIR", "1")
    if variant == "band":
        monkeypatch.setenv("PDB_JOIN_BAND", "1")   # the band plan at this size
    t = np.arange(n, dtype=np.float64) * 0.09
    v = np.ones(d) / np.sqrt(d)
    X = (t[:, None] * v[None, :] + 3.0).astype(np.float32)
    tau = 0.1
    ol, orr, od = oracle.sim_join(X, None, tau, self_join=True)
    xt = torch.from_numpy(X).cuda()
    r = patchdb.sim_join_device(xt, None, tau, self_join=True, sort=True,
                                dense=variant == "dense", tf32=variant == "tf32")
    l, rr, dd = (t_.cpu().numpy() for t_ in r.to_torch(xt.device))
    assert len(ol) >= n - 2
    assert np.array_equal(l, ol) and np.array_equal(rr, orr)
    assert np.array_equal(dd, od.astype(np.float32))


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_offsets_scales_dims(monkeypatch, seed):
    """Random shapes, dimensions, offsets far from the data's spread, scales
    and thresholds at distance quantiles, through a random screen variant:
    the pair set and distances equal the oracle's."""
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([1, 2, 3, 5, 8, 13, 24, 31, 64, 100, 128, 200]))
    nL, nR = int(rng.integers(50, 1500)), int(rng.integers(50, 1500))
    scale = float(10.0 ** rng.uniform(-4, 3))
    off = rng.normal(0, 1, d) * scale * float(10.0 ** rng.uniform(0, 3))
    L = (rng.random((nL, d)) * scale + off).astype(np.float32)
    near = L[rng.integers(0, nL, nR // 2)] + rng.normal(0, scale * 0.01, (nR // 2, d))
    R = np.concatenate([near, rng.random((nR - nR // 2, d)) * scale + off]).astype(np.float32)
    dd = np.sqrt(((L[:200, None, :].astype(np.float64) - R[None, :200]) ** 2).sum(-1))
    tau = float(np.quantile(dd, rng.uniform(0.001, 0.05)))
    if seed % 3 == 0:
        # points on a line far from its centre, neighbours 0.9 tau apart: the
        # copies' rounding errors line up along the line (worst case)
        v = rng.normal(0, 1, d)
        v /= np.linalg.norm(v)
        tau = 0.1 * scale
        t = np.arange(max(nL, nR), dtype=np.float64) * 0.09 * scale
        L = (off + t[:nL, None] * v).astype(np.float32)
        R = (off + t[:nR, None] * v + 0.05 * scale * v).astype(np.float32)
    variant = rng.choice(["default", "dense", "band", "tf32", "nofold"])
    if seed % 2:  # the grouped re-check (with the fp32 pre-filter when it applies)
        monkeypatch.setenv("PDB_K3_GROUPED", "2")
    if seed % 4 == 1:  # bf16 copies for band plans too
        monkeypatch.setenv("PDB_SCREEN_FP16", "0")
    if variant == "band":
        monkeypatch.setenv("PDB_JOIN_BAND", "1")
    if variant == "nofold":
        monkeypatch.setenv("PDB_NO_FOLD", "1")
    self_join = bool(rng.integers(0, 2))
    res = patchdb.sim_join(L, None if self_join else R, tau, self_join=self_join,
                           dense=variant == "dense", tf32=variant == "tf32")
    ol, orr, od = oracle.sim_join(L, None if self_join else R, tau, self_join=self_join, threads=4)
    _check(res, ol, orr, od)


def test_host_output_path_large():
    """The host API's pair output above 64 MB per array (config 5's
    distribution at 600k rows, ~22 M pairs): staged through the pinned ring
    in several chunks with threaded host copies (capi.cu d2h_large); equal
    to the device path's pairs."""
    x = workloads.config5(600_000)
    res = patchdb.sim_join(x, None, 0.01, self_join=True, sort=True)
    assert len(res.left) * 4 > (64 << 20)
    xt = torch.from_numpy(x).cuda()
    r = patchdb.sim_join_device(xt, None, 0.01, self_join=True, sort=True)
    want = [t.cpu().numpy() for t in r.to_torch(xt.device)]
    r.free()
    assert np.array_equal(res.left, want[0]) and np.array_equal(res.right, want[1])
    assert np.array_equal(res.dist, want[2])


def test_concurrent_host_threads():
    """Joins and featurization from four host threads at once (ctypes drops
    the GIL; each thread has its own stream, record cache and pinned
    read-back slot): every result equals the single-threaded one."""
    import threading
    xs = [workloads.config1(6000, seed=s) for s in range(4)]
    fr, _ = workloads.frames(40, 480, 640, seed=3)
    want = [patchdb.sim_join(x, None, 0.05, self_join=True, sort=True) for x in xs]
    want_f = patchdb.featurize_tiles(fr, 60, 80, 4, "joint")
    got, errs = [None] * 4, []

    def work(k):
        try:
            for _ in range(5):
                r = patchdb.sim_join(xs[k], None, 0.05, self_join=True, sort=True)
                f = patchdb.featurize_tiles(fr, 60, 80, 4, "joint")
                assert np.array_equal(f, want_f)
            got[k] = r
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert np.array_equal(w.left, g.left) and np.array_equal(w.right, g.right)
        assert np.array_equal(w.dist, g.dist)
