# K3 blocks per SM (PDB_K3_GRID, default 8; 4 resident at 64 registers)
for v in 4 8 12 16; do
  for w in c1 c3; do PDB_K3_GRID=$v timeout 300 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/k3g${v}_$w.log 2>&1; done
  PDB_K3_GRID=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config3 > gpurun_out/k3g${v}_c2.log 2>&1
  echo grid $v done
done
