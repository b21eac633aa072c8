"""Times pdb_featurize_join on pinned host frames (the bench's e2e call) and
prints a CUDA activity timeline of the last call.  Diagnostic only."""
import ctypes as C
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import _capi as capi  # noqa: E402
from paper_1812_07607_b200 import workloads  # noqa: E402

lib = capi.lib()
fr, _ = workloads.frames(1000, seed=2)
h = torch.from_numpy(fr).pin_memory()
o = capi.JoinOpts()


def call():
    pr = capi.Pairs()
    t0 = time.perf_counter()
    rc = lib.pdb_featurize_join(h.data_ptr(), 1000, 480, 640, 60, 80, 4, capi.PDB_HIST_JOINT, 0.05,
                                C.byref(o), None, C.byref(pr))
    t1 = time.perf_counter()
    assert rc == 0, capi.last_error()
    lib.pdb_pairs_free(C.byref(pr))
    return (t1 - t0) * 1e3


for _ in range(2):
    call()
print("ms", [round(call(), 2) for _ in range(4)])
if "--trace" in sys.argv:
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        call()
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs[-45:]:
        print(f"{e.time_range.start - t0:10.1f} dur {e.time_range.end - e.time_range.start:9.1f} {e.name[:70]}")
    cpu = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU),
                 key=lambda e: -(e.time_range.end - e.time_range.start))
    for e in cpu[:12]:
        print(f"CPU {e.name[:50]:50s} {e.time_range.end - e.time_range.start:9.1f} us")
