"""Repeats pdb_featurize_join_dev (K1 first-round count + PCA beside K1) and
checks every call's features and pairs against the first call's."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import _capi as capi, patchdb, workloads  # noqa: E402

n_calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lib = capi.lib()
for frames, seed in ((1000, 2), (257, 5), (130, 9)):
    fr, _ = workloads.frames(frames, 480, 640, seed=seed)
    d = torch.from_numpy(fr).cuda()
    feats = torch.empty(frames * 64, 64, device="cuda")
    o = capi.JoinOpts()
    o.flags = capi.PDB_JOIN_SELF | capi.PDB_JOIN_SORTED
    o.stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ref = None
    for it in range(n_calls):
        p = patchdb.DevicePairs()
        assert lib.pdb_featurize_join_dev(d.data_ptr(), frames, 480, 640, 60, 80, 4, 1, 0.05, C.byref(o),
                                          feats.data_ptr(), C.byref(p._p), C.byref(p.stats)) == 0
        got = [feats.cpu().numpy().copy()] + [t.cpu().numpy() for t in p.to_torch(d.device)]
        if ref is None:
            ref = got
        else:
            for a, b in zip(ref, got):
                assert np.array_equal(a, b), f"call {it} differs ({frames} frames)"
        p.free()
    print(f"{frames} frames: {n_calls} calls identical ({len(ref[1])} pairs)", flush=True)
