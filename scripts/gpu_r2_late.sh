#!/bin/bash
# one GPU: the late part's stages before the update start when its own classes are done
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_large.py -q -x > $O/late_tests.log 2>&1; echo "exit $?" >> $O/late_tests.log
for v in 1 2 3; do
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/late_bench_$v.json 2>/dev/null
done
CUDA_DEVICE_MAX_CONNECTIONS=32 SPNGD_NO_GRAPH=1 SPNGD_STEP_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > /dev/null 2> $O/late_trace.err
