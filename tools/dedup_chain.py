"""dedup on dependency chains (points 0.9 tau apart): device time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_07607_b200 import patchdb, workloads
for n in (3000, 30000):
    X = torch.from_numpy((np.arange(n, dtype=np.float32) * 0.09).reshape(-1, 1)).cuda()
    for k in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        rep_of, nr = patchdb.dedup_device(X, 0.1)
        torch.cuda.synchronize()
        if k == 2: print(f"chain n={n}: {1e3*(time.perf_counter()-t):.2f} ms reps={nr}")
fr, _ = workloads.frames(1000, 480, 640, seed=2)
X = patchdb.featurize_tiles(torch.from_numpy(fr).cuda(), 60, 80, 4, "joint")
for k in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    rep_of, nr = patchdb.dedup_device(X, 0.05)
    torch.cuda.synchronize()
    if k == 2: print(f"config-2 tiles: {1e3*(time.perf_counter()-t):.3f} ms reps={nr}")
