"""Seeded synthetic workloads for BASELINE.json's configs (libpdb_gen.so).

The paper's datasets are not available; like the
reference's own bench harness every workload is a seeded
synthetic stand-in with the configured shapes and value distributions.
Seeds: config 1 uses 0 (as BASELINE.json states); configs 2-5 are unseeded
there and use 2, 3, 4, 5.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _capi as capi


def _threads() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


def clusters(n: int, d: int, centres: int, sigma: float, l1_normalise: bool, seed: int,
             row_seed: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    x = out if out is not None else np.empty((n, d), dtype=np.float32)
    rs = seed if row_seed is None else row_seed
    rc = capi.gen().pdb_gen_clusters(capi.ptr(x), n, d, centres, sigma, int(l1_normalise), seed,
                                     rs, _threads())
    assert rc == 0
    return x


def uniform(n: int, d: int, seed: int) -> np.ndarray:
    x = np.empty((n, d), dtype=np.float32)
    capi.gen().pdb_gen_uniform(capi.ptr(x), n, d, seed, _threads())
    return x


def plant(L: np.ndarray, R: np.ndarray, frac: float, sigma: float, seed: int):
    """Config 3 planting; returns (left_idx, right_idx) of the planted pairs."""
    cap = int(L.shape[0] * frac * 2 + 1024)
    pl = np.empty(cap, dtype=np.int32)
    pr = np.empty(cap, dtype=np.int32)
    n = capi.gen().pdb_gen_plant(capi.ptr(L), L.shape[0], capi.ptr(R), R.shape[0], L.shape[1],
                                 frac, sigma, seed, capi.ptr(pl), capi.ptr(pr), cap)
    assert n <= cap
    return pl[:n].copy(), pr[:n].copy()


def simplex(n: int, d: int, centres: int, clustered: float, sigma: float, seed: int) -> np.ndarray:
    x = np.empty((n, d), dtype=np.float32)
    capi.gen().pdb_gen_simplex(capi.ptr(x), n, d, centres, clustered, sigma, seed, _threads())
    return x


def frames(F: int, H: int = 480, W: int = 640, *, block: int = 40, noise: int = 8,
           copy_noise: int = 4, period: int = 20, seed: int = 2, first: int = 0, out=None):
    """Config 2 frames first .. first+F-1 as [F, H, W, 3] uint8, and the
    source frame of each near-copy (-1 for originals).  ``out`` may be any
    writable [F, H, W, 3] uint8 numpy view (e.g. of pinned host memory)."""
    x = out if out is not None else np.empty((F, H, W, 3), dtype=np.uint8)
    src = np.empty(F, dtype=np.int64)
    rc = capi.gen().pdb_gen_frames(capi.ptr(x), first, F, H, W, block, noise, copy_noise, period,
                                   seed, capi.ptr(src), _threads())
    assert rc == 0
    return x, src


@dataclass(frozen=True)
class JoinConfig:
    name: str
    n: int
    d: int
    tau: float
    self_join: bool


CONFIG1 = JoinConfig("config1_selfjoin_20k_d64", 20_000, 64, 0.05, True)
CONFIG3 = JoinConfig("config3_cross_1M_d128", 1_048_576, 128, 0.02, False)
CONFIG5 = JoinConfig("config5_selfjoin_4M_d64", 4_194_304, 64, 0.01, True)


def config1(n: int = 20_000, seed: int = 0) -> np.ndarray:
    """200 Gaussian clusters (centres U[0,1]^64, sigma 0.02), L1-normalised."""
    return clusters(n, 64, 200, 0.02, True, seed)


def config3(n: int = 1_048_576, seed: int = 3, centres: int = 10_000):
    """L, R: 10,000-cluster mixture (sigma 0.01, unit cube), d=128, with 0.5%
    of L rows planted as R rows + 1e-3 N(0,1)."""
    R = clusters(n, 128, centres, 0.01, False, seed, row_seed=seed * 1000 + 1)
    L = clusters(n, 128, centres, 0.01, False, seed, row_seed=seed * 1000 + 2)
    pl, pr = plant(L, R, 0.005, 1e-3, seed)
    return L, R, pl, pr


def config5(n: int = 4_194_304, seed: int = 5) -> np.ndarray:
    """64-d simplex points: 20% in 50 clusters of sigma 1e-3, 80% Dirichlet(1)."""
    return simplex(n, 64, 50, 0.2, 1e-3, seed)


CONFIG2 = dict(frames=1000, H=480, W=640, tile_h=60, tile_w=80, bins=4, mode="joint",
               tau=0.05, seed=2)


def config4(n: int = 200_000, d: int = 2048, seed: int = 4, plant_frac: float = 0.005,
            plant_sigma: float = 0.2, device: str = "cpu", return_planted: bool = False):
    """Config 4: e = normalize(ReLU(P z)) stored as bf16, z ~ N(0,1)^d, P a
    fixed seeded d x d N(0,1)/sqrt(d) projection (torch's seeded CPU
    generator).  Independent ReLU'd projections sit near cosine ~0.3, so as
    stated the join would be empty; a fraction `plant_frac` of rows are
    therefore near-duplicates (z_i = z_src + plant_sigma * N(0,1)) to make
    the cos >= 0.95 parity check non-vacuous.  Returns a [n, d] torch bf16
    tensor on `device` (the product reads it; the oracle reads its uint16
    bits via .view(torch.int16)); with ``return_planted`` also the planted
    (row, source row) index pairs as int64 numpy arrays."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    P = torch.randn(d, d, generator=g) / d ** 0.5
    Z = torch.randn(n, d, generator=g)
    k = int(n * plant_frac)
    dst = src = torch.empty(0, dtype=torch.int64)
    if k:
        dst = torch.randperm(n, generator=g)[:k]
        src = torch.randint(0, n, (k,), generator=g)
        Z[dst] = Z[src] + plant_sigma * torch.randn(k, d, generator=g)
    P, Z = P.to(device), Z.to(device)
    out = torch.empty((n, d), dtype=torch.bfloat16, device=device)
    step = 16384
    for a in range(0, n, step):
        e = torch.relu(Z[a:a + step] @ P.T)
        e = e / e.norm(dim=1, keepdim=True).clamp_min(1e-30)
        out[a:a + step] = e.to(torch.bfloat16)
    if return_planted:
        return out, dst.numpy(), src.numpy()
    return out


def bf16_bits(t) -> np.ndarray:
    """uint16 bit patterns of a bf16 torch tensor (host numpy)."""
    import torch
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
