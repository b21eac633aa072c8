timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phase_ms']); print(d['e2e']['value'], d['e2e']['roofline']['frac'])"
for c in c1 c2; do timeout 300 python tools/join_sweep.py $c 2>&1 | tail -2; done
