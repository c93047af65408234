#!/bin/bash
# pair kernel with a dedicated MMA warp: parity + bench (+ implicit-im2col device time) + stage trace.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_large.py -q -x > $O/r2n_tests.log 2>&1; echo "exit $?" >> $O/r2n_tests.log
timeout 300 python scripts/gemm_micro.py > $O/r2n_micro.log 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2n_bench.json 2>$O/r2n_bench.err
make -s -C paper_2002_06015_b200 clean >/dev/null 2>&1
make -s -j16 -C paper_2002_06015_b200 TRACE=1 > $O/r2n_build.log 2>&1
SPNGD_NO_GRAPH=1 SPNGD_GEMM_TRACE=1 timeout 300 python scripts/syrk_one.py 1 > $O/r2n_pair_trace.log 2>&1
