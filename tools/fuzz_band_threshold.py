"""Joins in the size range the r02g rule moved onto the band plan (4,096 to
16,384 dense tiles on one GPU): random clustered / uniform / shifted data,
self and cross joins, default plan vs PDB_JOIN_BAND=0 (bit-identical sorted
output) and vs the brute-force oracle on sampled rows.
Usage: python tools/fuzz_band_threshold.py [n_cases]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 12
bad = 0
for c in range(n_cases):
    rng = np.random.default_rng(500 + c)
    d = int(rng.choice([8, 24, 32, 64, 100, 128]))
    self_join = bool(rng.integers(0, 2))
    nL = int(rng.integers(16_000, 34_000)) if self_join else int(rng.integers(9_000, 24_000))
    nR = nL if self_join else int(rng.integers(9_000, 24_000))
    kind = rng.choice(["clustered", "uniform", "shifted"])
    if kind == "clustered":
        L = workloads.clusters(nL, d, int(rng.integers(20, 400)), 0.02, True, 600 + c)
        tau = 0.05 / np.sqrt(64 / d)
    else:
        L = rng.random((nL, d), dtype=np.float32)
        if kind == "shifted":
            L = (L * 1e-2 + 50.0).astype(np.float32)
        dd = np.sqrt(((L[:300, None, :].astype(np.float64) - L[None, 300:600]) ** 2).sum(-1))
        tau = float(np.quantile(dd, 0.002))
    R = None if self_join else (L[rng.integers(0, nL, nR)] +
                                rng.normal(0, tau / 3, (nR, d))).astype(np.float32)
    Lt = torch.from_numpy(L).cuda()
    Rt = None if R is None else torch.from_numpy(R).cuda()
    outs = []
    for band in (None, "0"):
        if band is None:
            os.environ.pop("PDB_JOIN_BAND", None)
        else:
            os.environ["PDB_JOIN_BAND"] = band
        r = patchdb.sim_join_device(Lt, Rt, float(tau), self_join=self_join, sort=True)
        outs.append(([t.cpu().numpy() for t in r.to_torch(Lt.device)], r.stats.launches))
    os.environ.pop("PDB_JOIN_BAND", None)
    same = all(np.array_equal(a, b) for a, b in zip(outs[0][0], outs[1][0]))
    rows = np.unique(rng.integers(0, nL, 256))
    ol, orr, od = oracle.sim_join_rows(L, R, float(tau), rows, self_join=self_join)
    m = np.isin(outs[0][0][0], rows)
    ok = (np.array_equal(outs[0][0][0][m], ol) and np.array_equal(outs[0][0][1][m], orr) and
          np.array_equal(outs[0][0][2][m], od.astype(np.float32)))
    banded = outs[0][1] > outs[1][1]
    bad += (not same) or (not ok)
    print(f"case {c}: {kind:9s} d={d:3d} nL={nL} nR={nR} self={self_join} band={banded} "
          f"pairs={len(outs[0][0][0])} same_as_dense={same} oracle_rows_ok={ok}", flush=True)
print("failures", bad)
