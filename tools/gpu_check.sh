# Full GPU check: parity tests, smoke, bench, join sweeps over the configs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench.log
for c in c1 c2 c3s c4 c5:1048576; do echo "== $c"; timeout 300 python tools/join_sweep.py $c 2>&1 | tail -4; done
