#!/bin/bash
# precondition GEMMs on the 2-CTA kernel: parity tests + bench.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_large.py -q -x > $O/r2j_tests.log 2>&1; echo "exit $?" >> $O/r2j_tests.log
timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2j_bench.json 2>$O/r2j_bench.err
