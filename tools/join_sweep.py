"""Times the join on config-2 features (64,000 x 64 joint histograms) and
optionally other shapes; prints per-phase device times from pdb_join_stats."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c2":
    fr, _ = workloads.frames(1000, seed=2)
    X = patchdb.featurize_tiles(torch.from_numpy(fr).cuda(), 60, 80, 4, "joint")
    R, tau, self_join = None, 0.05, True
elif which == "c1":
    X = torch.from_numpy(workloads.config1()).cuda()
    R, tau, self_join = None, 0.05, True
elif which == "c3s":   # config-3 shaped, 1/4 size per side
    L, Rn, _, _ = workloads.config3(262144)
    X, R, tau, self_join = torch.from_numpy(L).cuda(), torch.from_numpy(Rn).cuda(), 0.02, False
elif which.startswith("c5"):   # config 5 (optionally scaled: c5:<n>)
    n5 = int(which.split(":")[1]) if ":" in which else 4_194_304
    X = torch.from_numpy(workloads.config5(n5)).cuda()
    R, tau, self_join = None, 0.01, True
elif which == "c4":
    X = workloads.config4(device="cuda")
    R, tau, self_join = None, 0.95, True
out = patchdb.DevicePairs()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
n = X.shape[0]
pairs = n * (n - 1) / 2 if self_join else n * R.shape[0]
for k in range(6):
    flush.zero_()
    torch.cuda.synchronize()
    if which == "c4":
        patchdb.cosine_join_bf16_device(X, R, tau, self_join=self_join, out=out, phase_times=True)
    else:
        patchdb.sim_join_device(X, R, tau, self_join=self_join, out=out,
                                tf32=os.environ.get("PDB_TF32") == "1", phase_times=True)
    st = out.stats
    if k >= 2:
        print(f"{which}: pairs={st.pairs} cand={st.candidates} tiles={st.tiles} prep={st.prep_ms:.3f} "
              f"screen={st.screen_ms:.3f} recheck={st.recheck_ms:.3f} ms  "
              f"{pairs / (st.screen_ms * 1e-3) / 1e9:.0f} Gpairs/s screen, "
              f"{pairs * 2 * X.shape[1] / (st.screen_ms * 1e-3) / 1e12:.1f} TFLOP/s", flush=True)
