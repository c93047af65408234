#!/bin/bash
# Split-K chunk sweep of the factor SYRK (L2 residency of the shared panels vs
# per-item overhead).  One bench line per chunk, no CPU leg, no e2e.
O=gpurun_out
for kc in default 4096 8192 16384; do
  if [ $kc = default ]; then unset SPNGD_KCHUNK; else export SPNGD_KCHUNK=$kc; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/kc_$kc.json 2> $O/kc_$kc.err
done
