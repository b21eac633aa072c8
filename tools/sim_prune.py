"""CPU simulation of the band plan's tile pruning: 2-D Morton keys of the two
principal projections vs adding the radial coordinate ||x - mu|| (as a
separate exact test or a 3-D key).  Counts kept 128x256 tiles of a
self-join (no error margins).  Usage: python tools/sim_prune.py c2|c5|c3"""
import sys, numpy as np, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_1812_07607_b200 import workloads
from oracle import oracle

def prune_counts(X, tau, self_join=True, BM=128, BN=256):
    n, d = X.shape
    mu = X[:256].mean(0)
    Xc = (X - mu).astype(np.float64)
    S = Xc[np.linspace(0, n - 1, 4096).astype(int)]
    C = S.T @ S
    w, V = np.linalg.eigh(C)
    U = V[:, ::-1][:, :2]
    P = Xc @ U
    r = np.linalg.norm(Xc, axis=1)
    out = {}
    def q(v, bits):
        lo, hi = np.percentile(v, 0.5), np.percentile(v, 99.5)
        return np.clip(((v - lo) / (hi - lo + 1e-30) * (1 << bits)).astype(int), 0, (1 << bits) - 1)
    def spread(x, k, dims):
        out = np.zeros_like(x)
        for b in range(k):
            out |= ((x >> b) & 1) << (b * dims)
        return out
    keys = {
        '2d6': spread(q(P[:, 0], 6), 6, 2) | (spread(q(P[:, 1], 6), 6, 2) << 1),
        '3d4': spread(q(P[:, 0], 4), 4, 3) | (spread(q(P[:, 1], 4), 4, 3) << 1) | (spread(q(r, 4), 4, 3) << 2),
        '2d6+r': (spread(q(P[:, 0], 6), 6, 2) | (spread(q(P[:, 1], 6), 6, 2) << 1)) * 4096.0 + r / r.max(),
        '3d5': spread(q(P[:, 0], 5), 5, 3) | (spread(q(P[:, 1], 5), 5, 3) << 1) | (spread(q(r, 5), 5, 3) << 2),
    }
    for name, k in keys.items():
        order = np.argsort(k, kind='stable')
        Ps, rs = P[order], r[order]
        nb, nt = (n + BM - 1) // BM, (n + BN - 1) // BN
        def boxes(B, m):
            bx = np.zeros((m, 6))
            for t in range(m):
                p = Ps[t * B:(t + 1) * B]; rr = rs[t * B:(t + 1) * B]
                bx[t] = [p[:, 0].min(), p[:, 0].max(), p[:, 1].min(), p[:, 1].max(), rr.min(), rr.max()]
            return bx
        a, b = boxes(BM, nb), boxes(BN, nt)
        g0 = np.maximum(0, np.maximum(a[:, None, 0] - b[None, :, 1], b[None, :, 0] - a[:, None, 1]))
        g1 = np.maximum(0, np.maximum(a[:, None, 2] - b[None, :, 3], b[None, :, 2] - a[:, None, 3]))
        gr = np.maximum(0, np.maximum(a[:, None, 4] - b[None, :, 5], b[None, :, 4] - a[:, None, 5]))
        keep2 = g0 ** 2 + g1 ** 2 <= tau ** 2
        keep3 = keep2 & (gr <= tau)
        if self_join:
            I = np.arange(nb)[:, None]; J = np.arange(nt)[None, :]
            tri = J >= (I >> 1)
            keep2 &= tri; keep3 &= tri
        out[name] = (int(keep2.sum()), int(keep3.sum()))
    return out

t = time.time()
which = sys.argv[1]
if which == 'c2':
    fr, _ = workloads.frames(1000, seed=2)
    X = oracle.featurize_tiles(fr, 60, 80, 4, 1)
    print('c2', X.shape, prune_counts(X, 0.05), time.time() - t)
elif which == 'c5':
    X = workloads.config5(262_144)
    print('c5/16', prune_counts(X, 0.01), time.time() - t)
elif which == 'c3':
    L, R, _, _ = workloads.config3(n=131072)
    print('c3/8 (self on L)', prune_counts(L, 0.02), time.time() - t)
