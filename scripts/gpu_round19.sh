#!/bin/bash
# Unrolled similarity kernel: the stale/step/kernel GPU tests, config 4 at B=256, the kernel under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest19.log 2>&1; echo "pytest exit $?" >> $O/pytest19.log
timeout 600 python scripts/stale_bench.py --batch 256 > $O/stale19_b256.json 2> $O/stale19_b256.err; echo "exit $?" >> $O/stale19_b256.err
timeout 400 ncu --set full --clock-control none -k regex:stat_distance -s 1 -c 1 -o $O/statdist19 -f python scripts/stale_bench.py --batch 32 --steps 3 > $O/ncu_statdist19.log 2>&1
