for c in c1 c2; do timeout 300 python tools/join_sweep.py $c 2>&1 | tail -2; done
timeout 300 python tools/join_sweep.py c5:1048576 2>&1 | tail -2
timeout 600 python -m pytest tests/test_join_gpu.py tests/test_cosine_gpu.py -q -x 2>&1 | tail -2
