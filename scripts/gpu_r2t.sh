#!/bin/bash
# vectorised split-K reduce; chunk vs the inverse chain's SM wait: step time per chunk (graphed), plus traces
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x > $O/r2t_tests.log 2>&1; echo "exit $?" >> $O/r2t_tests.log
for kc in default 2048 3072 4096 6144; do
  if [ $kc = default ]; then unset SPNGD_KCHUNK; else export SPNGD_KCHUNK=$kc; fi
  for v in 1 2; do
    timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2t_kc${kc}_$v.json 2>/dev/null
  done
  CUDA_DEVICE_MAX_CONNECTIONS=32 SPNGD_NO_GRAPH=1 SPNGD_STEP_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > /dev/null 2> $O/r2t_trace_kc$kc.err
done
