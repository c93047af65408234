#!/bin/bash
# repack with float4 loads: parity (step tests use repacked hw = 49 captures), bench, kernel time
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_large.py tests/test_gpu_step.py -q -x > $O/rep_tests.log 2>&1; echo "exit $?" >> $O/rep_tests.log
for v in 1 2 3; do
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/rep_bench_$v.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:repack --csv --log-file $O/rep_ncu.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-raw-e2e > $O/rep_ncu.log 2>&1
