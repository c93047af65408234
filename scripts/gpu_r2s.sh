#!/bin/bash
# critical path of the P=1 wave schedule: labelled events of an ungraphed step; hardware queue count
set -u
O=gpurun_out
mkdir -p $O
CUDA_DEVICE_MAX_CONNECTIONS=32 SPNGD_NO_GRAPH=1 SPNGD_STEP_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2s_trace32.json 2> $O/r2s_trace32.err
for v in 1 2; do
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2s_conn32_$v.json 2>/dev/null
timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2s_conn8_$v.json 2>/dev/null
done
