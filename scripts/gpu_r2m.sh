#!/bin/bash
# leaf with early release (3 publish buffers): parity + bench; then the trace build:
# pair-kernel stage anatomy and the leaf phases.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_large.py tests/test_gpu_step.py -q -x > $O/r2m_tests.log 2>&1; echo "exit $?" >> $O/r2m_tests.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2m_bench.json 2>$O/r2m_bench.err
make -s -C paper_2002_06015_b200 clean >/dev/null 2>&1
make -s -j16 -C paper_2002_06015_b200 TRACE=1 > $O/r2m_build.log 2>&1
SPNGD_NO_GRAPH=1 SPNGD_GEMM_TRACE=1 timeout 300 python scripts/syrk_one.py 1 > $O/r2m_pair_trace.log 2>&1
SPNGD_NO_GRAPH=1 SPNGD_GEMM_TRACE=1 timeout 300 python scripts/inv_one.py 1 > $O/r2m_leaf_trace.log 2>&1
