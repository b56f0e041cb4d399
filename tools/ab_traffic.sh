#!/bin/bash
# DRAM bytes + duration of one S16X2 GEMM launch (n=16384) per build (ncu metrics only)
Q="--no-apsp --no-configs --no-e2e --no-cpu-baseline --no-parity --no-variants --steps 2 --warmup 1"
for lib in "$@"; do
  BTAS_LIB=$lib python bench.py $Q > /dev/null 2>&1 || { echo "plain run failed for $lib"; exit 1; }
done
for lib in "$@"; do
  echo "== $lib"
  BTAS_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --kernel-name-base demangled -k regex:MixS16 -s 2 -c 1 python bench.py $Q 2>&1 | \
    grep -E "dram__bytes|gpu__time|hit_rate"
done
