#!/bin/bash
# A/B of libbtas_cuda.so builds (BTAS_LIB) on the accumulate-epilogue GEMM
# (FW bulk-pass shape) and Floyd-Warshall n=32768: bash tools/ab_epi.sh lib1.so lib2.so ...
for rep in 1 2; do
for lib in "$@"; do
  echo "== $lib"
  BTAS_LIB=$lib python tools/gemm_k_sweep.py 32768 1024,8192 2 plain,acc
  BTAS_LIB=$lib python tools/fw_sizes.py 32768
done
done
