"""Config-5 join repeated: screen passes, capacity and phase times per call."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_194_304
x = torch.from_numpy(workloads.config5(n)).cuda()
out = patchdb.DevicePairs()
for k in range(5):
    r = patchdb.sim_join_device(x, None, 0.01, self_join=True, phase_times=(k % 2 == 1), out=out)
    torch.cuda.synchronize()
    st = r.stats
    print(k, "pairs", r.count, "cand", st.candidates, "cap", st.candidate_capacity, "passes", st.screen_passes,
          "tiles", st.tiles, "ms", round(st.prep_ms, 1), round(st.screen_ms, 1), round(st.recheck_ms, 1), flush=True)
