#!/bin/bash
# four waves on the end-of-round build (per-class precondition parts, late part in the schedule)
set -u
O=gpurun_out
mkdir -p $O
for wv in default 3072,1536,1000 3072,1536,1100; do
  if [ $wv = default ]; then unset SPNGD_WAVES; else export SPNGD_WAVES=$wv; fi
  for v in 1 2; do
    timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/waves3_${wv//,/_}_$v.json 2>/dev/null
  done
done
