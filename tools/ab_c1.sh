# config 1: dense screen (default) vs the band plan's row order (PDB_JOIN_BAND=1),
# with and without the grouped re-check
line() { python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()}, d.get('pairs'), d.get('candidates'), d.get('tiles'))"; }
line default
PDB_JOIN_BAND=1 line band
PDB_JOIN_BAND=1 PDB_K3_GROUPED=2 line band_grouped
PDB_K3_GROUPED=2 line dense_grouped
PDB_JOIN_BAND=1 PDB_K3_GROUPED=2 PDB_K3_FILTER=0 line band_grouped_nofilter
