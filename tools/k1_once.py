"""One K1 launch on the config-2 frames (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07607_b200 import patchdb, workloads
fr, _ = workloads.frames(1000, seed=2)
d = torch.from_numpy(fr).cuda()
for _ in range(3):
    patchdb.featurize_tiles(d, 60, 80, 4, "joint")
torch.cuda.synchronize()
