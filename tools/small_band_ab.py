"""Dense vs band plan on small self-joins (PDB_JOIN_BAND=0/1, read per
call): config 1 (1 M pairs, clustered), the same rows shuffled, and sparse
outputs (uniform rows, few or no pairs) at 10k-40k rows.  Device time per
call (CUDA events, L2 flushed by a read before each call, median of 15)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

rng = np.random.default_rng(3)
cases = {
    "c1_20k_clustered": (workloads.config1(), 0.05),
    "uniform_20k_64d": (rng.random((20_000, 64), dtype=np.float32), 0.5),
    "uniform_40k_64d": (rng.random((40_000, 64), dtype=np.float32), 0.5),
    "uniform_12k_32d": (rng.random((12_000, 32), dtype=np.float32), 0.3),
    "c1like_40k": (workloads.clusters(40_000, 64, 400, 0.02, True, 9), 0.05),
}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
out = patchdb.DevicePairs()
for name, (X, tau) in cases.items():
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    row = [name]
    for band in ("0", "1"):
        os.environ["PDB_JOIN_BAND"] = band
        ts = []
        for k in range(18):
            sink.copy_(flush.view(torch.int64).sum())
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            st = patchdb.sim_join_device(Xd, None, tau, self_join=True, out=out).stats
            e.record()
            torch.cuda.synchronize()
            if k >= 3:
                ts.append(s.elapsed_time(e))
        ts.sort()
        row.append(f"band={band} {ts[len(ts)//2]*1e3:7.1f} us pairs={st.pairs} cand={st.candidates} tiles={st.tiles}")
    print(" | ".join(row), flush=True)
