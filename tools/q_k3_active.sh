# K3 with 16 blocks per SM, a quarter taking part when the candidates are few
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in c1 c3 c5; do timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/act_$w.log 2>&1; echo $w rc=$?; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config3 > gpurun_out/act_c2.log 2>&1; echo c2 rc=$?
