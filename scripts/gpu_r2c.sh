#!/bin/bash
# Ring experiment: 6-stage "B lo over A raw" ring (default) vs the 4-stage ring.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x > $O/r2c_tests.log 2>&1; echo "exit $?" >> $O/r2c_tests.log
for R in 4 6; do
  SPNGD_GEMM_RING=$R timeout 300 python scripts/gemm_micro.py > $O/r2c_micro_$R.log 2>&1
  SPNGD_GEMM_RING=$R timeout 300 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2c_bench_$R.json 2>$O/r2c_bench_$R.err
done
