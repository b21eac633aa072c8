"""The C restatement (oracle/pdb_oracle.c) against the reference's own
outputs: golden fixtures minted from the compiled reference, the known-answer
vectors of the reference's tests, and -- where oracle/_ref is built -- live
random cross-checks.  CPU only."""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io


def test_hist_golden_bit_exact():
    n = 0
    for name, fr, th, tw, b, want in golden_io.hist_cases():
        got = oracle.featurize_tiles(fr, th, tw, b, 0)
        assert got.shape == want.shape, name
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), name
        n += 1
    assert n >= 15


def test_hist_known_answers():
    # test_etl.cpp:226-256: solid (255,0,129), B=8 -> bins 7 / 8+0 / 16+4
    fr = np.empty((1, 8, 8, 3), np.uint8)
    fr[...] = (255, 0, 129)
    h = oracle.featurize_tiles(fr, 8, 8, 8, 0)[0]
    assert h[7] == 1.0 and h[8] == 1.0 and h[20] == 1.0 and h.sum() == 3.0
    # all-128, B=8 -> 1.0 at 4, 12, 20
    fr[...] = 128
    h = oracle.featurize_tiles(fr, 8, 8, 8, 0)[0]
    assert h[4] == h[12] == h[20] == 1.0 and h.sum() == 3.0
    # per-channel slices sum to 1 within 1e-6 (test_etl.cpp:237-242)
    rng = np.random.default_rng(0)
    fr = rng.integers(0, 256, (2, 12, 16, 3), dtype=np.uint8)
    h = oracle.featurize_tiles(fr, 12, 16, 8, 0)
    assert np.allclose(h.reshape(2, 3, 8).sum(-1), 1.0, atol=1e-6)


def test_hist_f32_golden():
    px, want = golden_io.f32_case()
    got = oracle.color_histogram(px, 8, 0)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_joint_histogram_restatement():
    # Restated joint mode: index (br*B + bg)*B + bb, L1 mass 1, and its
    # marginals equal the reference's per-channel histogram exactly.
    rng = np.random.default_rng(5)
    fr = rng.integers(0, 256, (2, 24, 32, 3), dtype=np.uint8)
    j = oracle.featurize_tiles(fr, 12, 16, 4, 1).reshape(-1, 4, 4, 4)
    p = oracle.featurize_tiles(fr, 12, 16, 4, 0).reshape(-1, 3, 4)
    cnt = np.rint(j * 192).astype(np.int64)
    pc = np.rint(p * 192).astype(np.int64)
    assert np.array_equal(cnt.sum((2, 3)), pc[:, 0])
    assert np.array_equal(cnt.sum((1, 3)), pc[:, 1])
    assert np.array_equal(cnt.sum((1, 2)), pc[:, 2])
    fr = np.zeros((1, 4, 4, 3), np.uint8)
    fr[..., 0], fr[..., 1], fr[..., 2] = 200, 70, 10   # bins 3, 1, 0 -> (3*4+1)*4+0 = 52
    j = oracle.featurize_tiles(fr, 4, 4, 4, 1)[0]
    assert j[52] == 1.0 and j.sum() == 1.0


def _ordered_pairs_of_self(li, ri):
    """Reference self-join output (ordered, incl. diagonal) -> i<j set."""
    m = li < ri
    return li[m], ri[m]


def test_join_golden_pairs_and_distances():
    for name, L, R, tau, sides, dist in golden_io.join_cases():
        side, (li, ri, probes) = next(iter(sides.items()))
        ol, orr, od = oracle.sim_join(L, R, tau, threads=4)
        assert np.array_equal(golden_io.canonical(ol, orr), golden_io.canonical(li, ri)), name
        # distances: bit-identical to the reference's euclidean()
        order = np.lexsort((ri, li))
        assert np.array_equal(od, dist[order]), name


def test_join_self_view_matches_reference_ordered_output():
    for name, L, R, tau, sides, dist in golden_io.join_cases():
        if name != "config1_3k":
            continue
        li, ri, _ = sides[2]
        a, b = _ordered_pairs_of_self(li, ri)
        ol, orr, _ = oracle.sim_join(L, None, tau, self_join=True, threads=4)
        assert np.array_equal(golden_io.canonical(ol, orr), golden_io.canonical(a, b))
        # the reference emits (i,i) for every row and both orientations
        assert len(li) == 2 * len(a) + L.shape[0]


def test_euclidean_known_answers():
    assert oracle.euclidean(np.array([0, 0], np.float32), np.array([3, 4], np.float32)) == 5.0
    a = np.array([1, 1], np.float32)
    b = np.array([2, 1], np.float32)
    assert oracle.euclidean(a, b) == 1.0   # inclusive radius case (test_index.cpp:330-342)


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built here")
def test_port_matches_reference_live():
    rng = np.random.default_rng(99)
    for d in (1, 3, 17, 64, 130):
        L = (rng.random((150, d)) * rng.choice([1e-3, 1.0, 1e3])).astype(np.float32)
        R = (L[rng.integers(0, 150, 90)] + rng.normal(0, 1e-3, (90, d))).astype(np.float32)
        dd = np.sqrt(((L[:, None, :].astype(np.float64) - R[None]) ** 2).sum(-1))
        tau = float(np.quantile(dd, 0.02))
        li, ri, _ = oracle.ref_sim_join(L, R, tau, 0)
        ol, orr, od = oracle.sim_join(L, R, tau, threads=2)
        assert np.array_equal(golden_io.canonical(ol, orr), golden_io.canonical(li, ri))
        for a, b, x in zip(ol[:50], orr[:50], od[:50]):
            assert x == oracle.ref_euclidean(L[a], R[b])
    fr = rng.integers(0, 256, (2, 30, 40, 3), dtype=np.uint8)
    for b in (2, 7, 13, 255, 256, 1000):
        assert np.array_equal(oracle.featurize_tiles(fr, 10, 8, b, 0).view(np.uint32),
                              oracle.ref_featurize_tiles(fr, 10, 8, b).view(np.uint32)), b


def test_dedup_restatement_matches_reference_golden():
    """orc_dedup (restated run_dedup) vs the reference's PlanNode::dedup
    membership and dedup_stream kept set, minted from oracle/_ref."""
    n_cases = 0
    for name, X, tau, rep_of, kept in golden_io.dedup_cases():
        got, nr = oracle.dedup(X, tau)
        assert np.array_equal(got, rep_of), name
        assert np.array_equal(np.flatnonzero(got == np.arange(X.shape[0])), kept), name
        assert nr == kept.shape[0]
        n_cases += 1
    assert n_cases >= 6


def test_dedup_restatement_live_vs_reference():
    if oracle.ref() is None:
        pytest.skip("oracle/_ref not built here")
    rng = np.random.default_rng(7)
    for n, d, tau in [(500, 2, 0.05), (800, 16, 0.9), (64, 1, 0.0)]:
        X = rng.random((n, d), dtype=np.float32)
        if tau == 0.0:
            X[::3] = X[0]  # exact duplicates at tau = 0
        got, nr = oracle.dedup(X, tau)
        want, nw = oracle.ref_dedup(X, tau)
        assert np.array_equal(got, want) and nr == nw
    assert oracle.ref_dedup(np.zeros((3, 2), np.float32), -1.0) == 1  # ConfigError


def test_nlj_within_and_q1_restatement_match_reference_golden():
    """The NLJ within contract is the brute-force pair set in (left, right)
    order; q1 is the self-join over whole-frame histograms in sim_join's
    emission order (probe = right, then ascending build id) minus same-frame
    pairs -- both pinned to the reference's own plan outputs."""
    for name, L, R, r, left, right in golden_io.nlj_cases():
        ol, orr, _ = oracle.sim_join(L, R, r)
        assert np.array_equal(ol, left) and np.array_equal(orr, right), name
    for name, fr, bins, tau, a, b in golden_io.q1_cases():
        H, W = fr.shape[1:3]
        h = oracle.featurize_tiles(fr, H, W, bins, 0)
        i, j, _ = oracle.sim_join(h, None, tau, self_join=True)
        ai = np.concatenate([i, j]).astype(np.int64)
        bj = np.concatenate([j, i]).astype(np.int64)
        order = np.lexsort((ai, bj))          # probe (right) order, then build id
        assert np.array_equal(ai[order], a) and np.array_equal(bj[order], b), name


# ---- the faster exact restatements used at full size ----------------------

def _same(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("d", [1, 2, 3, 7, 64, 128])
def test_pruned_and_rows_equal_plain_brute_force(d):
    from paper_1812_07607_b200 import workloads
    rng = np.random.default_rng(d)
    L = workloads.clusters(1500, d, 30, 0.02, False, d)
    R = np.concatenate([L[:400] + rng.normal(0, 0.01, (400, d)).astype(np.float32),
                        workloads.clusters(900, d, 30, 0.02, False, d + 1)]).astype(np.float32)
    for tau in (0.0, 0.02, 0.05, 0.3, 1e200):
        want = oracle.sim_join(L, R, tau, threads=4)
        assert _same(oracle.sim_join_pruned(L, R, tau, threads=3), want)
        rows = np.arange(0, 1500, 7)
        m = np.isin(want[0], rows)
        assert _same(oracle.sim_join_rows(L, R, tau, rows, threads=5),
                     (want[0][m], want[1][m], want[2][m]))
        ws = oracle.sim_join(L, None, tau, self_join=True, threads=4)
        assert _same(oracle.sim_join_pruned(L, None, tau, self_join=True), ws)


def test_pruned_edge_rows_and_boundaries():
    rng = np.random.default_rng(3)
    L = rng.random((700, 24), dtype=np.float32)
    R = L.copy()
    R[:, 0] += np.float32(0.25)            # distance exactly 0.25 for many rows
    L[5, 3] = np.nan
    L[6, 0] = np.inf
    R[7] = -np.inf
    L[8] = 3e30
    R[9] = 3e30
    R[10] = 3e30
    L[11] = 1e19
    R[12] = 1e19
    L[13, 2] = 7e12                          # beyond the grid: compared against all
    R[14, 2] = 7e12
    for tau in (0.25, np.nextafter(0.25, 0), 0.0, 1.5, float("inf")):
        want = oracle.sim_join(L, R, tau, threads=4)
        assert _same(oracle.sim_join_pruned(L, R, tau), want), tau
        assert _same(oracle.sim_join_rows(L, R, tau, np.arange(700)), want), tau
    assert len(oracle.sim_join_pruned(L, R, float("nan"))[0]) == 0
    with pytest.raises(RuntimeError):
        oracle.sim_join_pruned(L, R, -1.0)


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")
def test_pruned_equals_reference_sim_join():
    from paper_1812_07607_b200 import workloads
    x = workloads.config1(4000, seed=9)
    li, ri, _ = oracle.ref_sim_join(x, x, 0.05, 2)
    m = li < ri
    ol, orr, _ = oracle.sim_join_pruned(x, None, 0.05, self_join=True)
    assert np.array_equal(golden_io.canonical(ol, orr), golden_io.canonical(li[m], ri[m]))
