"""One config-5-distribution self-join (default 1M rows) for profiling K3."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
x = torch.from_numpy(workloads.config5(n)).cuda()
for _ in range(2):
    r = patchdb.sim_join_device(x, None, 0.01, self_join=True, phase_times=True)
    torch.cuda.synchronize()
    print(r.count, r.stats.candidates, r.stats.tiles, r.stats.screen_ms, r.stats.recheck_ms, r.stats.prep_ms)
    r.free()
