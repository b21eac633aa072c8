# one full ncu capture of K3 on config 1 (band plan), after the plain command exits 0
timeout 300 python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_recheck -s 3 -c 1 -o gpurun_out/prof_c1_recheck python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; echo ncu_rc=$?
