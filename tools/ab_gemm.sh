#!/bin/bash
# A/B of two builds of libbtas_cuda.so on the GEMM bench and the FW arm (same box, alternating)
Q="--no-apsp --no-configs --no-e2e --no-cpu-baseline --no-parity --steps 10"
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    BTAS_LIB=$lib python bench.py $Q 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); v=d.get('variants',{})
print('gemm', d['value'], d['roofline']['frac'], {k:(x['value'],x['frac']) for k,x in v.items()})"
    BTAS_LIB=$lib python bench.py --workload fw --steps 3 --no-e2e --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fw', d['value'], d['roofline']['frac'])"
  done
done
