L=paper_1701_04733_b200/_lib
for rep in 1 2; do
for lib in $L/libbtas_cuda_base.so $L/libbtas_cuda.so; do
  echo "== $lib"
  BTAS_LIB=$lib python tools/gemm_k_sweep.py 32768 1024,16384 2
  BTAS_LIB=$lib python tools/fw_sizes.py 32768
done
done
