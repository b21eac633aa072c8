"""Config-5 re-check A/B: PDB_K3_FILTER=1 (fp32 pre-filter, default) vs 0."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_194_304
x = torch.from_numpy(workloads.config5(n)).cuda()
for f in ("1", "0", "1", "0"):
    os.environ["PDB_K3_FILTER"] = f
    for ph in (True, False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        r = patchdb.sim_join_device(x, None, 0.01, self_join=True, phase_times=ph)
        ev[1].record()
        torch.cuda.synchronize()
        st = r.stats
        print(f"filter={f} phases={ph} total={ev[0].elapsed_time(ev[1]):.1f} ms pairs={r.count} "
              f"prep={st.prep_ms:.1f} screen={st.screen_ms:.1f} recheck={st.recheck_ms:.1f}", flush=True)
        r.free()
