#!/bin/bash
# same-box A/B: wave 0 prep (reduce/pi/unpack) inline on the main stream (default) vs beside the next SYRK
set -u
O=gpurun_out
mkdir -p $O
for v in 1 2 3; do
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/prep_w1_$v.json 2>/dev/null
  SPNGD_PREP_INLINE_WAVES=0 timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/prep_w0_$v.json 2>/dev/null
done
CUDA_DEVICE_MAX_CONNECTIONS=32 SPNGD_NO_GRAPH=1 SPNGD_STEP_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > /dev/null 2> $O/prep_w1_trace.err
