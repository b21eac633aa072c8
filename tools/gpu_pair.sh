timeout 120 python tools/join_sweep.py c2 2>&1 | tail -2
echo rc=$?
timeout 300 python -m pytest tests/test_join_gpu.py -q -x 2>&1 | tail -3
for c in c1 c3s c5:1048576; do timeout 120 python tools/join_sweep.py $c 2>&1 | tail -1; done
PDB_SCREEN_1SM=1 timeout 120 python tools/join_sweep.py c2 2>&1 | tail -1
