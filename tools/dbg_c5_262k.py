import sys, os, torch
sys.path.insert(0, '/root/repo')
from paper_1812_07607_b200 import patchdb, workloads
big = workloads.config5(262_144)
bt = torch.from_numpy(big).cuda()
for f16 in ("1", "0", "2"):
    os.environ["PDB_SCREEN_FP16"] = f16
    for _ in range(2):
        r = patchdb.sim_join_device(bt, None, 0.01, self_join=True, sort=True)
        st = r.stats
        print(f16, "passes", st.screen_passes, "cand", st.candidates, "cap", st.candidate_capacity, "pairs", st.pairs, "tiles", st.tiles, flush=True)
        r.free()
