#!/bin/bash
# 6-stage raw ring + separate B-lo ring GEMM: parity first, then the bench.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > $O/pytest_k10.log 2>&1; echo "pytest exit $?" >> $O/pytest_k10.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/bench10.json 2> $O/bench10.err; echo "exit $?" >> $O/bench10.err
