#!/bin/bash
# Round-2 measurement pass on one B200: GPU tests, default bench, every arm.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
python bench.py --workload apsp --n 512 > gpurun_out/r02_bench_apsp_n512.json 2>&1
python bench.py --workload fw --steps 3 > gpurun_out/r02_bench_fw_n32768.json 2>&1
for b in 1 2 4 8; do python bench.py --workload matvec --batch $b; done > gpurun_out/r02_bench_matvec.jsonl 2>&1
python bench.py --workload ewadd > gpurun_out/r02_bench_ewadd.json 2>&1
python bench.py --workload graph > gpurun_out/r02_bench_graph.json 2>&1
python bench.py --workload verify > gpurun_out/r02_bench_verify.json 2>&1
python bench.py --workload paths --steps 3 > gpurun_out/r02_bench_paths.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1
tail -3 gpurun_out/r02_pytest_gpu.log
