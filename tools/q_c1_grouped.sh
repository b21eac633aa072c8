# config 1 on the band plan: row-major vs grouped re-check (with / without the fp32 pre-filter)
for cfg in "1 1" "2 1" "2 0"; do set -- $cfg
  PDB_K3_GROUPED=$1 PDB_K3_FILTER=$2 timeout 300 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1_g$1_f$2.log 2>&1; echo g$1 f$2 rc=$?
done
