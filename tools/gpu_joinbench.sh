timeout 600 python -m pytest tests/test_bench_gpu.py -q -x 2>&1 | tail -3
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
  tail -1 gpurun_out/bench_$w.log | cut -c1-600
done
