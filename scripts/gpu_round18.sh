#!/bin/bash
# This session's kernel changes (fused snapshot rotation, warp-per-row im2col, 32-bit unpack_damp):
# full GPU suite, bench, config 4 at B=256, and the three kernels under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest18.log 2>&1; echo "pytest exit $?" >> $O/pytest18.log
timeout 600 python bench.py > $O/bench18.json 2> $O/bench18.err; echo "exit $?" >> $O/bench18.err
timeout 600 python scripts/stale_bench.py --batch 256 > $O/stale18_b256.json 2> $O/stale18_b256.err; echo "exit $?" >> $O/stale18_b256.err
timeout 400 ncu --set full --clock-control none -k regex:im2col -c 1 -o $O/im2col18 -f python scripts/raw_step.py > $O/ncu_im2col18.log 2>&1
timeout 400 ncu --set full --clock-control none -k regex:unpack_damp -c 1 -o $O/unpack18 -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_unpack18.log 2>&1
timeout 400 ncu --set full --clock-control none -k regex:stat_distance -s 1 -c 1 -o $O/statdist18 -f python scripts/stale_bench.py --batch 32 --steps 3 > $O/ncu_statdist18.log 2>&1
