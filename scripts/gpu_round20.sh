#!/bin/bash
# Flat float4 similarity kernel: the stale/step/kernel GPU tests, config 4 at B=256, the kernel under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest20.log 2>&1; echo "pytest exit $?" >> $O/pytest20.log
timeout 600 python scripts/stale_bench.py --batch 256 > $O/stale20_b256.json 2> $O/stale20_b256.err; echo "exit $?" >> $O/stale20_b256.err
timeout 400 ncu --set full --clock-control none -k regex:stat_distance -s 1 -c 1 -o $O/statdist20 -f python scripts/stale_bench.py --batch 32 --steps 3 > $O/ncu_statdist20.log 2>&1
