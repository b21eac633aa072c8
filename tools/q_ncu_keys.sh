# one full ncu capture of k_band_keys on config 3 (d = 128, 1M rows per side), after the plain command exits 0
timeout 300 python tools/timeline_join.py c3 --plain > gpurun_out/keys_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_band_keys -s 2 -c 1 -o gpurun_out/prof_keys python tools/timeline_join.py c3 --plain > gpurun_out/ncu_keys.log 2>&1; echo ncu_rc=$?
