timeout 60 python tools/hist_sweep.py 2>&1 | head -1
timeout 120 python -m pytest tests/test_hist_gpu.py -q -x 2>&1 | tail -1
