#!/bin/bash
# Wide (3 x 64-k, one two-plane TMA box per operand) vs narrow (4 x 32-k) engine ring.
set -u
O=gpurun_out
mkdir -p $O
for R in 4 6; do
  SPNGD_GEMM_RING=$R timeout 300 python scripts/gemm_micro.py > $O/r2d_micro_$R.log 2>&1
  SPNGD_GEMM_RING=$R timeout 300 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2d_bench_$R.json 2>$O/r2d_bench_$R.err
done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r2d_tests.log 2>&1; echo "exit $?" >> $O/r2d_tests.log
