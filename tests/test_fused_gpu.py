"""pdb_featurize_join_dev: featurize + self-join in one call, the band plan's
centre and directions computed on K1's first round while K1 still runs
(join.cu run_featurize_join_dev).  Features must be bit-identical to
pdb_featurize_tiles_dev and the pair set identical to pdb_sim_join_dev's
(only the screened tiles may differ) -- and to the oracle."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1812_07607_b200 import _capi as capi, patchdb, workloads

pytestmark = pytest.mark.gpu


def _run(fr, th, tw, B, mode, tau, fused, flags=0):
    lib = capi.lib()
    d = torch.from_numpy(fr).cuda()
    n, H, W = fr.shape[:3]
    tiles = n * (H // th) * (W // tw)
    D = lib.pdb_hist_dim(B, mode)
    feats = torch.empty(tiles, D, device="cuda")
    o = capi.JoinOpts()
    o.flags = capi.PDB_JOIN_SELF | flags
    o.stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = patchdb.DevicePairs()
    if fused:
        rc = lib.pdb_featurize_join_dev(d.data_ptr(), n, H, W, th, tw, B, mode, tau, C.byref(o),
                                        feats.data_ptr(), C.byref(p._p), C.byref(p.stats))
    else:
        rc = lib.pdb_featurize_tiles_dev(d.data_ptr(), n, H, W, th, tw, B, mode, feats.data_ptr(),
                                         o.stream)
        assert rc == 0
        rc = lib.pdb_sim_join_dev(feats.data_ptr(), tiles, feats.data_ptr(), tiles, D, tau,
                                  C.byref(o), C.byref(p._p), C.byref(p.stats))
    assert rc == 0, capi.last_error()
    l, r, dd = (t.cpu().numpy() for t in p.to_torch(d.device))
    k = np.lexsort((r, l))
    return feats.cpu().numpy(), l[k], r[k], dd[k], p.stats


@pytest.mark.parametrize("frames,reserve", [(1000, "1"), (300, "0"), (300, "3")])
def test_fused_matches_separate_calls(monkeypatch, frames, reserve):
    monkeypatch.setenv("PDB_FJ_RESERVE", reserve)  # read once per process: first value sticks
    fr, _ = workloads.frames(frames, 480, 640, seed=2)
    a = _run(fr, 60, 80, 4, 1, 0.05, True)
    b = _run(fr, 60, 80, 4, 1, 0.05, False)
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1:4], b[1:4]):
        assert np.array_equal(x, y)
    assert len(a[1]) > 10
    assert a[4].pairs == b[4].pairs


def test_fused_against_oracle_and_fallbacks(monkeypatch):
    """The oracle's pairs on a 150-frame set (9,600 tiles: above the band
    plan's size threshold); the dense and no-overlap fallbacks
    (PDB_JOIN_BAND=0, PDB_FUSED_PCA=0) give the same."""
    fr, _ = workloads.frames(150, 480, 640, seed=7)
    feats, l, r, dd, st = _run(fr, 60, 80, 4, 1, 0.05, True)
    ol, orr, od = oracle.sim_join(feats, None, 0.05, self_join=True)
    assert np.array_equal(l, ol) and np.array_equal(r, orr)
    assert np.array_equal(dd, od.astype(np.float32))
    for env in ("PDB_JOIN_BAND", "PDB_FUSED_PCA"):
        monkeypatch.setenv(env, "0")
        g = _run(fr, 60, 80, 4, 1, 0.05, True)
        assert np.array_equal(g[1], l) and np.array_equal(g[2], r)
        monkeypatch.delenv(env)


def test_fused_rejects_sharding():
    lib = capi.lib()
    fr, _ = workloads.frames(4, 480, 640, seed=1)
    d = torch.from_numpy(fr).cuda()
    feats = torch.empty(4 * 64, 64, device="cuda")
    o = capi.JoinOpts()
    o.shard_index, o.shard_count = 0, 2
    p = patchdb.DevicePairs()
    rc = lib.pdb_featurize_join_dev(d.data_ptr(), 4, 480, 640, 60, 80, 4, 1, 0.05, C.byref(o),
                                    feats.data_ptr(), C.byref(p._p), C.byref(p.stats))
    assert rc != 0


@pytest.mark.parametrize("B,mode", [(2, 1), (4, 0)])
def test_fused_other_histograms(B, mode):
    """K1 variants without the first-round signal (per-channel histograms) and
    the 8-bin joint one: the PCA then waits for K1, same pairs either way."""
    fr, _ = workloads.frames(200, 480, 640, seed=9)
    tau = 0.05 if mode == 1 else 0.03
    a = _run(fr, 60, 80, B, mode, tau, True)
    b = _run(fr, 60, 80, B, mode, tau, False)
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1:4], b[1:4]):
        assert np.array_equal(x, y)
