set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 120 python tools/measure_tf32_peak.py > gpurun_out/peaks.log 2>&1; echo peaks_rc=$?
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/bench.log | tail -3
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/prof_screen python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_tiles -s 2 -c 1 -o gpurun_out/prof_hist python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1; echo ncu3_rc=$?
ls -la gpurun_out
