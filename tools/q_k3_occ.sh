# K3 register/occupancy variants (build_exp/libpdb_cuda_{A,B,C}.so vs the product library)
for v in base A B C; do
  if [ $v = base ]; then unset PDB_CUDA_LIB; else export PDB_CUDA_LIB=$PWD/build_exp/libpdb_cuda_$v.so; fi
  for w in c1 c3 c5; do timeout 600 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/occ_${v}_$w.log 2>&1; echo $v $w rc=$?; done
done
