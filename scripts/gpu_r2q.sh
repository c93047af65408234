#!/bin/bash
# inverse-recursion and refinement GEMMs on the 2-CTA kernel: parity + bench (pair on / off) + config-5 sweep.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_large.py tests/test_gpu_stale.py -q -x > $O/r2q_tests.log 2>&1; echo "exit $?" >> $O/r2q_tests.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2q_bench.json 2>$O/r2q_bench.err
SPNGD_NO_PAIR=1 timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2q_bench_nopair.json 2>$O/r2q_bench_nopair.err
timeout 900 python scripts/inverse_sweep.py > $O/r2q_sweep.json 2>$O/r2q_sweep.err
