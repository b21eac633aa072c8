for i in 1 2 3; do python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()}, d['clocks']['reasons'])"; done
bash tools/ab_lines.sh 2>&1 | grep -E "^c2|^c3|^c1"
