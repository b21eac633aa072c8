# K3 blocks per SM with the adaptive participation (PDB_K3_BPS, default 16)
for v in 16 24 32; do
  for w in c1 c3; do PDB_K3_BPS=$v timeout 300 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bps${v}_$w.log 2>&1; done
  PDB_K3_BPS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config3 > gpurun_out/bps${v}_c2.log 2>&1
  PDB_K3_BPS=$v timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bps${v}_c5.log 2>&1
  echo bps $v done
done
