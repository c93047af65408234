#!/bin/bash
# ncu --set full of the other hot kernels of the current build (one launch each).
O=gpurun_out
mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
SPNGD_NO_OVERLAP=1 timeout 600 ncu --set full --clock-control none -k regex:base_chol_inv -s 20 -c 1 -o $O/leaf -f $B > $O/ncu_leaf.log 2>&1
SPNGD_NO_OVERLAP=1 timeout 600 ncu --set full --clock-control none -k "regex:gemm_tf32x3_kernel<8" -c 1 -o $O/precond -f $B > $O/ncu_precond.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:im2col -c 1 -o $O/im2col -f python scripts/raw_step.py > $O/ncu_im2col.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:unpack_damp -c 1 -o $O/unpack -f $B > $O/ncu_unpack.log 2>&1
