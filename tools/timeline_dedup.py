"""GPU timeline of one dedup call over the config-2 tiles (diagnostic)."""
import os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_join import _gen  # noqa: E402
from paper_1812_07607_b200 import patchdb  # noqa: E402
X, _ = _gen("dedup")
x = torch.from_numpy(X).cuda()
for _ in range(3):
    patchdb.dedup_device(x, 0.05)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    patchdb.dedup_device(x, 0.05)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} dur {e.time_range.end - e.time_range.start:8.1f} {e.name[:70]}")
