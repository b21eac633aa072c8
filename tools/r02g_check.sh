nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
for w in c1 c3 c5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
done
