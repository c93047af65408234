#!/bin/bash
# 2-CTA 256x256 SYRK vs the single-CTA engine.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > $O/r2g_kernels.log 2>&1; echo "exit $?" >> $O/r2g_kernels.log
for P in 0 1; do
  if [ $P = 1 ]; then export SPNGD_NO_PAIR=1; else unset SPNGD_NO_PAIR; fi
  timeout 300 python scripts/gemm_micro.py > $O/r2g_micro_nopair$P.log 2>&1
  timeout 300 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2g_bench_nopair$P.json 2>$O/r2g_bench_nopair$P.err
done
unset SPNGD_NO_PAIR
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_large.py tests/test_gpu_stale.py -q -x > $O/r2g_step.log 2>&1; echo "exit $?" >> $O/r2g_step.log
