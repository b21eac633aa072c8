"""GPU activity timeline (CUPTI via torch.profiler) of the config-2 device
step: featurize -> join.  Prints every kernel / memcpy / memset of the last
step with start offsets and durations, so launch gaps and host round trips
show up.  Diagnostic only."""
import ctypes as C
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import _capi as capi  # noqa: E402
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

lib = capi.lib()
fr, _ = workloads.frames(1000, seed=2)
d = torch.from_numpy(fr).cuda()
feats = torch.empty((64000, 64), device="cuda")
stream = torch.cuda.current_stream()
sptr = C.c_void_p(stream.cuda_stream)
pairs = patchdb.DevicePairs()
opts = capi.JoinOpts()
opts.flags = capi.PDB_JOIN_SELF
opts.stream = sptr


def step():
    torch.cuda.nvtx.range_push("step")
    assert lib.pdb_featurize_tiles_dev(d.data_ptr(), 1000, 480, 640, 60, 80, 4, capi.PDB_HIST_JOINT,
                                       feats.data_ptr(), sptr) == 0
    assert lib.pdb_sim_join_dev(feats.data_ptr(), 64000, feats.data_ptr(), 64000, 64, 0.05,
                                C.byref(opts), C.byref(pairs._p), C.byref(pairs.stats)) == 0
    torch.cuda.nvtx.range_pop()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
# last step: from the last histogram kernel on
last = max(i for i, e in enumerate(evs) if "hist" in e.name)
t0 = evs[last].time_range.start
prev_end = t0
for e in evs[last:]:
    s, t = e.time_range.start, e.time_range.end
    print(f"{s - t0:9.1f} us  gap {s - prev_end:7.1f}  dur {t - s:8.1f}  {e.name[:90]}")
    prev_end = t
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and
       e.name.startswith("cuda")]
cpu.sort(key=lambda e: e.time_range.start)
print("--- runtime API calls (last 40)")
for e in cpu[-40:]:
    print(f"{e.time_range.start - t0:9.1f} us  dur {e.time_range.end - e.time_range.start:8.1f}  {e.name}")
