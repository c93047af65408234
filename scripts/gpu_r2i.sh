#!/bin/bash
# pair threshold (n = 147, 256, 512 join the 2-CTA SYRK): factor tests + bench.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x > $O/r2i_tests.log 2>&1; echo "exit $?" >> $O/r2i_tests.log
timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2i_bench.json 2>$O/r2i_bench.err
