#!/bin/bash
# Wave-boundary sweep of the overlapped schedule (SPNGD_WAVES, larger Kronecker
# dimension thresholds, largest first).  One bench line each, no CPU leg, no e2e.
O=gpurun_out
i=0
for wv in "3072,1536" "3072,1536,768" "3072,1536,768,384" "3072,2048,1024,512" "3072,1024"; do
  SPNGD_WAVES=$wv timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/wv_$i.json 2> $O/wv_$i.err
  echo "$wv" > $O/wv_$i.cfg
  i=$((i+1))
done
