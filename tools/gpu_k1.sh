for v in 0 8 10 11 9; do echo v=$v; PDB_K1_VARIANT=$v timeout 60 python tools/hist_sweep.py 2>&1 | head -1; done
timeout 300 python -m pytest tests/test_hist_gpu.py -q -x 2>&1 | grep -v "^  File\|^Extension\|^Thread\|^Current" | tail -25
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_hist_joint_rows8 -s 3 -c 1 -o gpurun_out/prof_k1rows8 python tools/hist_sweep.py > gpurun_out/ncu_k1.log 2>&1; echo ncu_rc=$?
