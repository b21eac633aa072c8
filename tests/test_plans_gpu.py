"""Plans routed onto the B200 join: PlanNode::nl_join with
a within predicate, and the q1 near-duplicate-frame plan, against the
reference's own plan outputs (tests/golden/nlj_golden.npz)."""

import numpy as np
import pytest

from paper_1812_07607_b200 import patchdb
from tests import golden_io

pytestmark = pytest.mark.gpu


def _patches(X, first_id):
    return [patchdb.Patch(first_id + k, X[k], (X.shape[1],)) for k in range(X.shape[0])]


def test_nl_join_within_matches_reference_order():
    for name, L, R, r, left, right in golden_io.nlj_cases():
        lp, rp = _patches(L, 1), _patches(R, 1 << 32)
        got = patchdb.nl_join_within(lp, rp, r)
        assert [(a.patch_id - 1, b.patch_id - (1 << 32)) for a, b in got] == \
            list(zip(left.tolist(), right.tolist())), name


def test_nl_join_within_edges():
    a = patchdb.Patch(1, np.zeros(2, np.float32), (2,))
    b = patchdb.Patch(2, np.zeros(3, np.float32), (3,))
    with pytest.raises(patchdb.DimensionMismatchError):
        patchdb.nl_join_within([a], [b], 1.0)
    assert patchdb.nl_join_within([], [b], 1.0) == []
    assert patchdb.nl_join_within([a], [a], -1.0) == []


def test_q1_matches_reference_plan():
    for name, fr, bins, tau, a, b in golden_io.q1_cases():
        ga, gb = patchdb.q1_duplicate_frames(fr, bins, tau)
        assert np.array_equal(ga, a) and np.array_equal(gb, b), name
