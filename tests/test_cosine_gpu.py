"""Config-4 cosine join over bf16 rows (restated; the reference has no
cosine predicate): the pair set equals the restated fp64 oracle
(oracle/pdb_oracle.c orc_cosine_join_bf16) exactly."""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1812_07607_b200 import patchdb, workloads
from tests import golden_io

pytestmark = pytest.mark.gpu


def _check(res, ol, orr, oc):
    assert np.array_equal(golden_io.canonical(res.left, res.right), golden_io.canonical(ol, orr))
    order = np.lexsort((res.right, res.left))
    assert np.array_equal(res.dist[order], oc.astype(np.float32))


@pytest.mark.parametrize("d", [16, 64, 100, 128, 300, 2048])
def test_cosine_small_vs_oracle(d):
    x = workloads.config4(3000, d=d, seed=d, plant_frac=0.05, plant_sigma=0.15)
    b = workloads.bf16_bits(x)
    res = patchdb.cosine_join_bf16(b, None, 0.95, self_join=True)
    ol, orr, oc = oracle.cosine_join_bf16(b, None, 0.95, self_join=True)
    assert len(ol) > 10
    _check(res, ol, orr, oc)
    cr = patchdb.cosine_join_bf16(b[:1700], b[1200:], 0.9)
    ol, orr, oc = oracle.cosine_join_bf16(b[:1700], b[1200:], 0.9)
    _check(cr, ol, orr, oc)


def test_cosine_edge_rows_and_thresholds():
    rng = np.random.default_rng(5)
    a = np.abs(rng.standard_normal((400, 96))).astype(np.float32)
    a[3] = 0.0                       # zero row: never matches
    a[4, 7] = np.inf                 # non-finite row: never matches
    a[5] = -a[6]                     # anti-parallel pair
    b = (a.view(np.uint32) >> 16).astype(np.uint16)
    for c in (0.99, 0.5, 0.0, -0.5, -1.0):
        res = patchdb.cosine_join_bf16(b, None, c, self_join=True)
        ol, orr, oc = oracle.cosine_join_bf16(b, None, c, self_join=True)
        _check(res, ol, orr, oc)
        assert 3 not in res.left and 3 not in res.right and 4 not in res.left
    with pytest.raises(patchdb.ConfigError):
        patchdb.cosine_join_bf16(b, None, 1.5, self_join=True)


def test_config4_full_size_sampled_rows():
    """200,000 x 2048 bf16 (config 4): the device join, checked exactly on
    sampled row blocks against the restated fp64 oracle (the planted
    near-duplicates: test_fullsize_gpu.test_config4_planted_pairs_found)."""
    x = workloads.config4(device="cuda")
    out = patchdb.cosine_join_bf16_device(x, None, 0.95, self_join=True, sort=True)
    l, r, c = (t.cpu().numpy() for t in out.to_torch(x.device))
    assert out.stats.pairs == len(l) > 500
    b = workloads.bf16_bits(x)
    for r0 in (0, 123_456, 199_900):
        ol, orr, oc = oracle.cosine_join_bf16(b, None, 0.95, self_join=True, rows=(r0, r0 + 48))
        m = (l >= r0) & (l < r0 + 48)
        assert np.array_equal(l[m], ol) and np.array_equal(r[m], orr)
        assert np.array_equal(c[m], oc.astype(np.float32))
