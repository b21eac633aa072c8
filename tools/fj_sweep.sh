# fused featurize->join (PCA beside K1): partial blocks (sample = 64 x blocks rows)
for b in 64 16 8; do echo "pca_blocks=$b"; PDB_FJ_PCA_BLOCKS=$b timeout 300 python tools/fused_ab.py 2>&1 | grep -E "us pairs"; done
PDB_FJ_PCA_BLOCKS=16 timeout 300 python tools/fused_ab.py --timeline 2>&1 | grep -E "k_hist|k_col_mean|k_pca|k_wait|k_band_keys|k_screen"
