"""Times K1 variants on config-2 frames resident in HBM (L2 flushed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

fr, _ = workloads.frames(1000, seed=2)
d = torch.from_numpy(fr).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode, bins in (("joint", 4), ("per_channel", 4), ("per_channel", 8), ("joint", 8)):
    ts = []
    for k in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        patchdb.featurize_tiles(d, 60, 80, bins, mode)
        e.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(s.elapsed_time(e))
    ms = sum(ts) / len(ts)
    print(f"{mode:12s} B={bins}: {ms*1e3:8.1f} us  {921.6e6/(ms*1e-3)/1e9:7.1f} GB/s read", flush=True)
