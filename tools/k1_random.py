"""K1 (joint B = 4, 60x80 tiles) on the config-2 frames and on uniform-random
frames of the same shape, frames resident in HBM, L2 flushed by a 256 MB
read before each launch: the counting uses lane-private counters, so the
time should not depend on the pixel content."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

fr, _ = workloads.frames(1000, seed=2)
cases = {
    "config2": torch.from_numpy(fr).cuda(),
    "uniform_random": torch.randint(0, 256, fr.shape, dtype=torch.uint8, device="cuda",
                                    generator=torch.Generator(device="cuda").manual_seed(7)),
    "constant": torch.full(fr.shape, 77, dtype=torch.uint8, device="cuda"),
}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
for name, d in cases.items():
    ts = []
    for k in range(13):
        sink.copy_(flush.view(torch.int64).sum())  # read-flush (clean lines)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        patchdb.featurize_tiles(d, 60, 80, 4, "joint")
        e.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(s.elapsed_time(e))
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{name:15s} median {med*1e3:7.1f} us  min {ts[0]*1e3:7.1f} us  "
          f"{937.984e6/(med*1e-3)/1e9:7.1f} GB/s algorithmic", flush=True)
