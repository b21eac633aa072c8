"""Cost of the first library call in a fresh process (CUDA context, module
load, pool creation) vs a warm call."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.perf_counter()
from paper_1812_07607_b200 import _capi as capi, patchdb
import numpy as np
t1 = time.perf_counter()
x = np.random.default_rng(0).random((20000, 24), dtype=np.float32)
y = np.random.default_rng(1).random((20000, 24), dtype=np.float32)
for k in range(4):
    t = time.perf_counter()
    r = patchdb.sim_join(x, y, 0.1)
    print(f"call {k}: {1e3*(time.perf_counter()-t):.1f} ms ({len(r)} pairs)", flush=True)
print(f"import {1e3*(t1-t0):.0f} ms")
