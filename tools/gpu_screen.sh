timeout 900 python -m pytest tests/test_join_gpu.py tests/test_cosine_gpu.py tests/test_dropin_gpu.py -q -x 2>&1 | tail -2
for c in c1 c2 c3s c4 c5:1048576; do timeout 300 python tools/join_sweep.py $c 2>&1 | tail -2; done
PDB_TF32=1 timeout 300 python tools/join_sweep.py c2 2>&1 | tail -1
