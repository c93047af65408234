#!/bin/bash
# im2col with four columns per lane in flight: parity, raw-input step, ncu of the kernel
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "raw" > $O/r2z_tests.log 2>&1; echo "exit $?" >> $O/r2z_tests.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $O/r2z_bench.json 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:im2col_kernel -c 1 -o $O/r2z_im2col python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/r2z_ncu.log 2>&1
