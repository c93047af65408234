#!/bin/bash
# same-box A/B: precondition stage kernel choice by wave cost vs always 2-CTA
set -u
O=gpurun_out
mkdir -p $O
for v in 1 2 3; do
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/pre2_wave_$v.json 2>/dev/null
  SPNGD_PRE_PAIR_ALWAYS=1 timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/pre2_always_$v.json 2>/dev/null
done
