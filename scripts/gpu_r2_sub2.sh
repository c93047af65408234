#!/bin/bash
# host-input sub-waves: 4 vs 8 vs 2 layer groups
set -u
O=gpurun_out
mkdir -p $O
for n in 2 4 8; do
  for v in 1 2; do
    SPNGD_SUBWAVES=$n timeout 600 python bench.py --steps 5 --e2e-steps 10 --no-cpu-baseline --no-raw-e2e > $O/sub2_${n}_$v.json 2>/dev/null
  done
done
