for v in 0 1 2 3; do echo v=$v; PDB_HIST_VARIANT=$v timeout 60 python tools/hist_sweep.py 2>&1 | head -1; done
for v in 0 2; do PDB_HIST_VARIANT=$v timeout 120 python -m pytest tests/test_hist_gpu.py -q -x 2>&1 | tail -1; done
