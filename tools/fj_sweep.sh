# fused featurize->join (PCA beside K1): partial blocks (sample = 64 x blocks rows)
for b in 64 32 48; do echo "pca_blocks=$b"; PDB_FJ_PCA_BLOCKS=$b timeout 300 python tools/fused_ab.py 2>&1 | grep -E "fused"; done
