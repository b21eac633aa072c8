import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
t = time.perf_counter()
rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
from paper_1812_07607_b200 import _capi as capi, patchdb
lib = capi.lib()
t0 = time.perf_counter()
print("device_count", lib.pdb_device_count(), f"{1e3*(time.perf_counter()-t0):.0f} ms", flush=True)
x = np.random.default_rng(0).random((2000, 24), dtype=np.float32)
for k in range(3):
    t = time.perf_counter()
    patchdb.featurize_tiles(np.zeros((1, 64, 64, 3), np.uint8), 8, 8, 4, "joint")
    print(f"featurize call {k}: {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
for k in range(3):
    t = time.perf_counter()
    patchdb.sim_join(x, x, 0.1)
    print(f"join call {k}: {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
