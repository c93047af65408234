#!/bin/bash
# Similarity kernel: idle warps skip their atomics. Stale + kernel GPU tests, the kernel under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_stale.py tests/test_gpu_kernels.py -m gpu -q > $O/pytest21.log 2>&1; echo "pytest exit $?" >> $O/pytest21.log
timeout 300 ncu --set full --clock-control none -k regex:stat_distance -s 1 -c 1 -o $O/statdist21 -f python scripts/stale_bench.py --batch 32 --steps 3 > $O/ncu_statdist21.log 2>&1
