import ctypes as C, time, sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1812_07607_b200 import _capi as capi, patchdb, workloads
lib = capi.lib()
x = workloads.config1()
hx = torch.from_numpy(x).pin_memory()
o = capi.JoinOpts(); o.flags = capi.PDB_JOIN_SELF
def e2e():
    pr = capi.Pairs()
    t0 = time.perf_counter()
    assert lib.pdb_sim_join(hx.data_ptr(), x.shape[0], hx.data_ptr(), x.shape[0], 64, 0.05, C.byref(o), C.byref(pr)) == 0
    t1 = time.perf_counter()
    lib.pdb_pairs_free(C.byref(pr))
    t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3
for _ in range(3): e2e()
print("e2e call ms, free ms:", [tuple(round(v, 3) for v in e2e()) for _ in range(5)])
dx = torch.from_numpy(x).cuda()
od = capi.JoinOpts(); od.flags = capi.PDB_JOIN_SELF; od.stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = patchdb.DevicePairs()
def dev():
    torch.cuda.synchronize(); t0 = time.perf_counter()
    assert lib.pdb_sim_join_dev(dx.data_ptr(), x.shape[0], dx.data_ptr(), x.shape[0], 64, 0.05, C.byref(od), C.byref(p._p), C.byref(p.stats)) == 0
    torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
for _ in range(3): dev()
print("dev call ms:", [round(dev(), 3) for _ in range(5)])
