"""Dedup (the paper's near-duplicate grouping) on the B200:
pdb_dedup / pdb_dedup_dev and the object API against the reference's own
PlanNode::dedup / dedup_stream outputs (tests/golden/dedup_golden.npz) and
the C restatement."""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1812_07607_b200 import patchdb, workloads
from tests import golden_io

pytestmark = pytest.mark.gpu


def test_golden_membership_host_and_device():
    for name, X, tau, rep_of, kept in golden_io.dedup_cases():
        g = patchdb.dedup(X, tau)
        assert np.array_equal(g.rep_of, rep_of), name
        assert np.array_equal(g.reps, kept), name
        dev, nr = patchdb.dedup_device(torch.from_numpy(np.ascontiguousarray(X)).cuda(), tau)
        assert nr == kept.shape[0] and np.array_equal(dev.cpu().numpy(), rep_of), name


def test_members_in_arrival_order():
    X, tau = next((X, t) for n, X, t, _, _ in golden_io.dedup_cases() if n == "test_query_6pts")
    g = patchdb.dedup(X, tau)
    assert [list(m) for m in g.members] == [[0, 1, 3], [2, 4], [5]]


def test_object_api_matches_reference_test_query():
    """test_query.cpp:331-368: group sizes, labels and lineage parents."""
    patchdb.reset_patch_ids()
    pts = [(1, 0.00, 0.00, "a"), (2, 0.01, 0.00, "b"), (3, 1.00, 1.00, "a"),
           (4, 0.00, 0.02, "a"), (5, 1.01, 1.00, "c"), (6, 5.00, 5.00, "d")]
    items = [patchdb.Patch(pid, np.array([x, y], np.float32), (2,), {"label": lab})
             for pid, x, y, lab in pts]
    out = patchdb.dedup_groups(items, 0.1)
    assert [p.lineage[0].source for p in out] == [1, 3, 6]
    assert out[0].meta["group_size"] == 3 and out[2].meta["group_size"] == 1
    assert out[0].meta["group_labels"] == ["a", "b"]
    assert out[1].meta["group_labels"] == ["a", "c"]
    again = patchdb.dedup_groups(out, 0.1)
    assert len(again) == 3
    kept = list(patchdb.dedup_stream(items, 0.1))
    assert [p.patch_id for p in kept] == [1, 3, 6]


def test_errors_and_degenerate():
    with pytest.raises(patchdb.ConfigError):
        patchdb.dedup(np.zeros((3, 2), np.float32), -0.1)
    g = patchdb.dedup(np.zeros((0, 4), np.float32), 0.1)
    assert g.reps.size == 0 and g.rep_of.size == 0
    g = patchdb.dedup(np.zeros((5, 4), np.float32), 0.0)   # all identical at tau 0
    assert list(g.reps) == [0] and list(g.rep_of) == [0] * 5
    a = patchdb.Patch(1, np.zeros(2, np.float32), (2,))
    b = patchdb.Patch(2, np.zeros(3, np.float32), (3,))
    with pytest.raises(patchdb.MixedDimensionError):
        patchdb.dedup_groups([a, b], 0.1)
    with pytest.raises(patchdb.ShapeError):
        list(patchdb.dedup_stream([patchdb.Patch(3, np.zeros(0, np.float32), (0,))], 0.1))


@pytest.mark.parametrize("case", ["config1_full", "config2_4000", "chain_1d", "nan_rows",
                                  "chain_30k", "chain_branchy", "chain_then_clique"])
def test_against_restatement(case):
    if case == "config1_full":          # 20,000 rows, ~1e6 tau-graph edges
        X, tau = workloads.config1(), 0.05
    elif case == "config2_4000":
        fr, _ = workloads.frames(63, 480, 640, seed=2)
        X, tau = oracle.featurize_tiles(fr, 60, 80, 4, 1)[:4000], 0.05
    elif case == "chain_1d":            # a long dependency chain: points 0.9 tau apart
        X, tau = (np.arange(3000, dtype=np.float32) * 0.09).reshape(-1, 1), 0.1
    elif case == "chain_30k":           # decided by the sequential tail (k_dedup_tail) in chunks
        X, tau = (np.arange(30000, dtype=np.float32) * 0.09).reshape(-1, 1), 0.1
    elif case == "chain_then_clique":   # tail items with more edges than the tail's stage holds
        chain = (np.arange(200, dtype=np.float32) * 0.09).reshape(-1, 1)
        rng = np.random.default_rng(4)
        clique = (chain[-1, 0] + 0.09 + rng.random((42000, 1)) * 0.01).astype(np.float32)
        X, tau = np.concatenate([chain, clique]).astype(np.float32), 0.1
    elif case == "chain_branchy":       # chains with several lower neighbours per item
        rng = np.random.default_rng(9)
        X = np.cumsum(rng.random((12000, 2), dtype=np.float32) * 0.04, axis=0).astype(np.float32)
        tau = 0.1
    else:
        rng = np.random.default_rng(3)
        X = rng.random((1500, 8), dtype=np.float32)
        X[::7, 3] = np.nan
        tau = 0.4
    want, nr = oracle.dedup(X, tau)
    g = patchdb.dedup(X, tau)
    assert g.reps.size == nr
    assert np.array_equal(g.rep_of, want)
