timeout 300 python tools/k1_random.py 2>&1 | tail -4
for b in 0 1; do PDB_JOIN_BAND=$b timeout 300 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1_band$b.log 2>&1; echo band$b rc=$?; done
