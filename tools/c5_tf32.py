"""Config-5 join: bf16 vs tf32 screen copies (phase times, candidates)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07607_b200 import patchdb, workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_194_304
x = torch.from_numpy(workloads.config5(n)).cuda()
out = patchdb.DevicePairs()
for tf32 in (False, True, False, True):
    for ph in (False, True):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = patchdb.sim_join_device(x, None, 0.01, self_join=True, tf32=tf32, out=out, phase_times=ph)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        st = r.stats
        print(f"tf32={tf32} phases={ph} wall={t*1e3:.1f} ms pairs={st.pairs} cand={st.candidates} "
              f"prep={st.prep_ms:.1f} screen={st.screen_ms:.1f} recheck={st.recheck_ms:.1f} passes={st.screen_passes}", flush=True)
