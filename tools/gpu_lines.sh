# Every bench line (device + e2e + CPU baseline) after a change.
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo c2 rc=$?
for w in c1 c3 c4 c5 dedup; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
done
