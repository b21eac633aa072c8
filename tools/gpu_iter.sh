set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for a in 0 1; do PDB_HIST_ATOMS=$a timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_atoms$a.log 2>&1; echo rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_atoms$a.log').read().strip().splitlines()[-1]); print('atoms=$a', d['value'], d['phase_ms'], d['roofline_all'][0]['frac'], d['roofline_all'][1]['frac'], d['e2e']['ms_per_step'], d['pairs'], d['candidates'])"; done
