"""CPU simulation: Morton keys over the top D principal projections (D = 2..6,\nbits per dimension) with D-dimensional tile boxes; counts kept 128x256 tiles\nof a self-join.  Usage: python tools/sim_prune_nd.py c2|c5|c3"""
import sys, numpy as np, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_1812_07607_b200 import workloads
from oracle import oracle
def run(X, tau, BM=128, BN=256):
    n, d = X.shape
    mu = X[:256].mean(0)
    Xc = (X - mu).astype(np.float64)
    S = Xc[np.linspace(0, n - 1, 4096).astype(int)]
    w, V = np.linalg.eigh(S.T @ S)
    U = V[:, ::-1][:, :6]
    P = Xc @ U
    def q(v, bits):
        lo, hi = np.percentile(v, 0.5), np.percentile(v, 99.5)
        return np.clip(((v - lo) / (hi - lo + 1e-30) * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    def morton(cols, bits):
        k = np.zeros(n, np.int64); D = len(cols)
        for i, c in enumerate(cols):
            for b in range(bits):
                k |= ((c >> b) & 1) << (b * D + i)
        return k
    res = {}
    for D, bits in ((2, 6), (3, 6), (4, 6), (4, 5), (6, 4)):
        k = morton([q(P[:, i], bits) for i in range(D)], bits)
        o = np.argsort(k, kind='stable'); Ps = P[o]
        nb, nt = (n + BM - 1) // BM, (n + BN - 1) // BN
        def bx(B, m):
            lo = np.array([Ps[t*B:(t+1)*B, :D].min(0) for t in range(m)]); hi = np.array([Ps[t*B:(t+1)*B, :D].max(0) for t in range(m)])
            return lo, hi
        al, ah = bx(BM, nb); bl, bh = bx(BN, nt)
        g2 = np.zeros((nb, nt))
        for i in range(D):
            g = np.maximum(0, np.maximum(al[:, None, i] - bh[None, :, i], bl[None, :, i] - ah[:, None, i]))
            g2 += g * g
        keep = g2 <= tau * tau
        tri = np.arange(nt)[None, :] >= (np.arange(nb)[:, None] >> 1)
        res[(D, bits)] = int((keep & tri).sum())
    return res
w = sys.argv[1]
if w == 'c2':
    fr, _ = workloads.frames(1000, seed=2); X = oracle.featurize_tiles(fr, 60, 80, 4, 1); print('c2', run(X, 0.05))
elif w == 'c5':
    print('c5/16', run(workloads.config5(262_144), 0.01))
elif w == 'c3':
    L, R, _, _ = workloads.config3(n=131072); print('c3/8', run(L, 0.02))
