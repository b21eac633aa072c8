# Band-plan check: full GPU suite, then the bench lines that use the join.
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2 rc=$?
tail -1 gpurun_out/bench_c2.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phase_ms']); print(d['roofline_all'][1])"
for w in c1 c3 c5 dedup; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
  tail -1 gpurun_out/bench_$w.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['unit'], d['ms_per_step'], d.get('phase_ms'), d['roofline'].get('frac'), d['roofline'].get('tiles_screened'), d['roofline'].get('tiles_dense'), d.get('pairs'))"
done
