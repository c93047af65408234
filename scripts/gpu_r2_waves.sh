#!/bin/bash
# wave boundaries: move the 1024-class layers (layer3 1x1 convs) into wave 1
set -u
O=gpurun_out
mkdir -p $O
for wv in default 3072,1000 3072,1100,600; do
  if [ $wv = default ]; then unset SPNGD_WAVES; else export SPNGD_WAVES=$wv; fi
  for v in 1 2; do
    timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/waves_${wv//,/_}_$v.json 2>/dev/null
  done
done
