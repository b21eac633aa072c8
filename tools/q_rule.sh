# after the single-GPU band threshold change: all GPU tests, then the c1 line
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --workload c1 --steps 10 --warmup 3 > gpurun_out/rule_c1.log 2>&1; echo c1 rc=$?
timeout 300 python tools/small_band_ab.py 2>&1 | tail -6
