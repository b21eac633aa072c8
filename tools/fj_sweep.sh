# fused featurize->join (PCA beside K1) vs separate calls; K1's reserved SMs
for r in 0 1 2; do echo "reserve=$r"; PDB_FJ_RESERVE=$r timeout 300 python tools/fused_ab.py 2>&1 | grep -E "us pairs"; done
PDB_FJ_RESERVE=0 timeout 300 python tools/fused_ab.py --timeline 2>&1 | grep -E "k_hist|k_col_mean|k_pca|k_wait|k_band_keys|k_screen"
