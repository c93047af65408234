#!/bin/bash
# wave boundaries x split-K chunk: step time (graphed) and a trace per config
set -u
O=gpurun_out
mkdir -p $O
for wv in default 3072,1536,1000 3072,1536,1000,600; do
for kc in default 4096; do
  if [ $kc = default ]; then unset SPNGD_KCHUNK; else export SPNGD_KCHUNK=$kc; fi
  if [ $wv = default ]; then unset SPNGD_WAVES; else export SPNGD_WAVES=$wv; fi
  tag=w${wv//,/_}_kc$kc
  for v in 1 2; do
    timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2u_${tag}_$v.json 2>/dev/null
  done
  CUDA_DEVICE_MAX_CONNECTIONS=32 SPNGD_NO_GRAPH=1 SPNGD_STEP_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > /dev/null 2> $O/r2u_trace_$tag.err
done
done
