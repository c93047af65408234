#!/bin/bash
# Fused snapshot rotation: stale parity tests, config 4 at B=256 on one GPU, and the similarity kernel under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stale.py tests/test_gpu_step.py -m gpu -q > $O/pytest16.log 2>&1; echo "pytest exit $?" >> $O/pytest16.log
timeout 600 python scripts/stale_bench.py --batch 256 > $O/stale16_b256.json 2> $O/stale16_b256.err; echo "exit $?" >> $O/stale16_b256.err
timeout 600 ncu --set full --clock-control none -k regex:stat_distance -s 1 -c 1 -o $O/statdist -f python scripts/stale_bench.py --batch 32 --steps 3 > $O/ncu_statdist.log 2>&1
