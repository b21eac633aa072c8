"""Config-2 step: pdb_featurize_join_dev (PCA on a prefix sample beside K1)
vs pdb_featurize_tiles_dev + pdb_sim_join_dev; same pairs, device times."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import _capi as capi, patchdb, workloads  # noqa: E402

lib = capi.lib()
fr, _ = workloads.frames(1000, 480, 640, seed=2)
d = torch.from_numpy(fr).cuda()
n, H, W = fr.shape[:3]
th, tw, B, mode, tau = 60, 80, 4, 1, 0.05
tiles = n * (H // th) * (W // tw)
D = lib.pdb_hist_dim(B, mode)
feats = torch.empty(tiles, D, device="cuda")
s = torch.cuda.current_stream()
o = capi.JoinOpts()
o.flags = capi.PDB_JOIN_SELF
o.stream = C.c_void_p(s.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def fused(p):
    assert lib.pdb_featurize_join_dev(d.data_ptr(), n, H, W, th, tw, B, mode, tau, C.byref(o),
                                      feats.data_ptr(), C.byref(p._p), C.byref(p.stats)) == 0, capi.last_error()


def split(p):
    assert lib.pdb_featurize_tiles_dev(d.data_ptr(), n, H, W, th, tw, B, mode, feats.data_ptr(),
                                       C.c_void_p(s.cuda_stream)) == 0
    assert lib.pdb_sim_join_dev(feats.data_ptr(), tiles, feats.data_ptr(), tiles, D, tau, C.byref(o),
                                C.byref(p._p), C.byref(p.stats)) == 0


def pairs_of(p):
    l, r, dd = (t.cpu().numpy() for t in p.to_torch(d.device))
    k = np.lexsort((r, l))
    return l[k], r[k], dd[k]


res = {}
for name, fn in (("split", split), ("fused", fused), ("split", split), ("fused", fused)):
    p = patchdb.DevicePairs()
    ts = []
    for it in range(25):
        flush.amax()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(p)
        e1.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    res[name] = pairs_of(p)
    print(name, f"{np.mean(ts)*1e3:.1f} us", "pairs", p.count, "cand", p.stats.candidates, "tiles",
          p.stats.tiles, flush=True)
for a, b in zip(res["split"], res["fused"]):
    assert np.array_equal(a, b)
print("pairs identical")

if "--timeline" in sys.argv:
    from torch.profiler import ProfilerActivity, profile
    p = patchdb.DevicePairs()
    fused(p)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.cuda._sleep(1_000_000)
        fused(p)
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"{e.time_range.start - t0:10.1f} us  dur {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
