for f in 1 0 2; do
  echo "fp16=$f"
  PDB_SCREEN_FP16=$f python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()}, d.get('pairs'), d.get('candidates'))"
  for w in c3 c5; do PDB_SCREEN_FP16=$f python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()}, d.get('pairs'), d.get('candidates'))"; done
done
