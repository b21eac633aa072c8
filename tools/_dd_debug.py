import sys, os, subprocess; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import oracle
from paper_1812_07607_b200 import patchdb
import torch
n = int(os.environ.get("N", 5000))
X, tau = (np.arange(n, dtype=np.float32) * 0.09).reshape(-1, 1), 0.1
ol, orr, od = oracle.sim_join(X, None, tau, self_join=True)
s2 = set(zip(ol.tolist(), orr.tolist()))
xt = torch.from_numpy(X).cuda()
for kw in (dict(), dict(dense=True), dict(tf32=True)):
    r = patchdb.sim_join_device(xt, None, tau, self_join=True, sort=True, **kw)
    l, rr, d = (t.cpu().numpy() for t in r.to_torch(xt.device))
    s1 = set(zip(l.tolist(), rr.tolist()))
    print(os.environ.get("TAG",""), kw, "gpu", len(s1), "oracle", len(s2), "missing", sorted(s2 - s1)[:4], "cand", r.stats.candidates, "tiles", r.stats.tiles)
