#!/bin/bash
# Leaf / GEMM-round anatomy with the clock64 trace build (box-local rebuild).
set -u
O=gpurun_out
mkdir -p $O
make -s -C paper_2002_06015_b200 clean >/dev/null 2>&1
make -s -j16 -C paper_2002_06015_b200 TRACE=1 > $O/r2k_build.log 2>&1
SPNGD_NO_GRAPH=1 SPNGD_GEMM_TRACE=1 timeout 300 python scripts/inv_one.py 2 > $O/r2k_trace.log 2>&1
