# K2: folded -||y||^2/2 (default) vs epilogue subtraction (PDB_NO_FOLD=1)
for v in 0 1; do echo "no_fold=$v"; PDB_NO_FOLD=$v bash tools/ab_lines.sh 2>&1; done
