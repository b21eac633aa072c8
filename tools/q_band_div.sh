# work units per SM of band-plan screens (PDB_BAND_DIV, default 8)
for v in 4 8 16 32; do
  PDB_BAND_DIV=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config3 > gpurun_out/div${v}_c2.log 2>&1
  for w in c1 c3; do PDB_BAND_DIV=$v timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/div${v}_$w.log 2>&1; done
  echo div $v done
done
