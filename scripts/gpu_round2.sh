#!/bin/bash
# Second pass: the new step-mode GPU tests, a full capture of the whole
# factor SYRK launch (phase-serial schedule), and the 2-GPU bench line.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_stale.py -m gpu -x -q > $O/pytest_step.log 2>&1; echo "pytest exit $?" >> $O/pytest_step.log
SPNGD_NO_OVERLAP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -c 1 \
  -o $O/factor_syrk_full -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $O/ncu_full2.log 2>&1; echo "ncu full exit $?" >> $O/ncu_full2.log
