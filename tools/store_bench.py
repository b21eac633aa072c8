"""Frame source throughput: a config-2-sized store (1000 frames 480x640,
segmented lossless clips of 32, written by the reference's VideoStore::ingest)
decoded by libpdb_cuda and featurized by K1, vs the reference's own
VideoStore::scan (oracle/_ref) on the same file.  Diagnostic / profiles only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_1812_07607_b200 import patchdb, workloads  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
path = "/tmp/pdb_store_c2.pdb"
fr, _ = workloads.frames(F, 480, 640, seed=2)
t0 = time.perf_counter()
assert oracle.ref_store_write(fr, path, 2, 0, 32) == 0
print(f"reference ingest: {time.perf_counter() - t0:.2f} s, {os.path.getsize(path) / 1e6:.1f} MB")
st = patchdb.VideoStore.open(path)
for _ in range(2):
    st.featurize(60, 80, 4, "joint")
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    feats = st.featurize(60, 80, 4, "joint")
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"B200 decode+K1: {t * 1e3:.1f} ms -> {F / t:.0f} frames/s ({os.cpu_count()} host threads)")
t0 = time.perf_counter()
arr = st.scan_array()
t_dec = time.perf_counter() - t0
print(f"  decode only: {t_dec * 1e3:.1f} ms -> {F / t_dec:.0f} frames/s")
k = min(F, 64)
t0 = time.perf_counter()
ref = oracle.ref_store_scan(path, F, 480, 640, 0, k)
t_ref = (time.perf_counter() - t0) * F / k
print(f"reference VideoStore::scan: {F / t_ref:.0f} frames/s (first {k} frames, 1 thread)")
assert np.array_equal(ref, arr[:k])
want = oracle.featurize_tiles(arr[:8], 60, 80, 4, 1)
assert np.array_equal(feats[:8 * 64].cpu().numpy().view(np.uint32), want.view(np.uint32))
print("parity ok")
