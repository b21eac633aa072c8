"""Times K1 (joint 4x4x4, config 2) under PDB_K1_GROUP = 1, 2, 4 on the
config-2 frames and on uniform-random frames, L2 flushed, and checks each
variant bit-exact against the oracle on sampled frames."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
from paper_1812_07607_b200 import patchdb, workloads
from oracle import oracle
fr, _ = workloads.frames(1000, seed=2)
rng = np.random.default_rng(0)
rnd = rng.integers(0, 256, fr.shape, dtype=np.uint8)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for name, x in (("config2", fr), ("uniform", rnd)):
    d = torch.from_numpy(x).cuda()
    ts = []
    for k in range(12):
        torch.cuda.synchronize(); flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); h = patchdb.featurize_tiles(d, 60, 80, 4, "joint"); e.record()
        torch.cuda.synchronize()
        if k >= 4: ts.append(s.elapsed_time(e))
    hh = h.cpu().numpy()
    for f in ((0, 333, 999) if os.environ["PDB_K1_GROUP"] != "0" and os.environ.get("PDB_K1_EPI") != "0" else ()):
        want = oracle.featurize_tiles(x[f:f+1], 60, 80, 4, 1)
        assert np.array_equal(hh[f*64:(f+1)*64].view(np.uint32), want.view(np.uint32)), (name, f)
    ms = sorted(ts)[len(ts)//2]
    out[name] = {"us": ms * 1e3, "GBps": 937984e3 / (ms * 1e-3) / 1e9}
print(json.dumps(out))
""" % ROOT
# each argument: comma-separated env settings, e.g. PDB_K1_GROUP=0,PDB_K1_STAGES=4
for spec in sys.argv[1:] or ["PDB_K1_GROUP=1"]:
    env = dict(os.environ, PDB_K1_GROUP="1")
    for kv in spec.split(","):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(spec, r.stdout.strip() or r.stderr[-2000:], flush=True)
