"""GPU activity timeline (CUPTI via torch.profiler) of one join-only bench
workload (default c3; c2 = the config-2 tile histograms): every kernel of the last call with start offsets and
durations.  Diagnostic only.  Usage: python tools/timeline_join.py [c3|c5|c1]"""
import ctypes as C
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_join import JOINS, _gen  # noqa: E402
from paper_1812_07607_b200 import _capi as capi  # noqa: E402
from paper_1812_07607_b200 import patchdb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
plain = "--plain" in sys.argv  # no profiler (for ncu)
if which == "c2":  # the config-2 tile histograms (bench.py's join)
    from paper_1812_07607_b200 import workloads  # noqa: E402
    fr, _ = workloads.frames(1000, 480, 640, seed=2)
    cfg = dict(self_join=True, tau=0.05)
    L, R = patchdb.featurize_tiles(fr, 60, 80, 4, "joint"), None
else:
    cfg = JOINS[which]
    L, R = _gen(which)
Ld = torch.from_numpy(L).cuda()
Rd = Ld if R is None else torch.from_numpy(R).cuda()
lib = capi.lib()
stream = torch.cuda.current_stream()
opts = capi.JoinOpts()
opts.flags = (capi.PDB_JOIN_SELF if cfg["self_join"] else 0) | \
    (capi.PDB_JOIN_PHASE_TIMES if "--phase" in sys.argv else 0)
opts.stream = C.c_void_p(stream.cuda_stream)
pairs = patchdb.DevicePairs()


def call():
    assert lib.pdb_sim_join_dev(Ld.data_ptr(), Ld.shape[0], Rd.data_ptr(), Rd.shape[0], Ld.shape[1],
                                float(cfg["tau"]), C.byref(opts), C.byref(pairs._p),
                                C.byref(pairs.stats)) == 0


for _ in range(2):
    call()
torch.cuda.synchronize()
if plain:
    sys.exit(0)
head = "--headstart" in sys.argv  # a ~0.5 ms spin first, so the host enqueues ahead of the device
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if head:
        torch.cuda._sleep(1_000_000)
    call()
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = t0
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    print(f"{s - t0:10.1f} us  gap {s - prev:8.1f}  dur {t - s:9.1f}  {e.name[:80]}")
    prev = t
print("tiles", pairs.stats.tiles, "pairs", pairs.count, "candidates", pairs.stats.candidates,
      "ms", pairs.stats.prep_ms, pairs.stats.screen_ms, pairs.stats.recheck_ms)
