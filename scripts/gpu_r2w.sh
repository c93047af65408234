#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "wave_schedule or failed or singular or host" > $O/r2w_tests.log 2>&1; echo "exit $?" >> $O/r2w_tests.log
for v in 1 2 3; do
  SPNGD_NO_OVERLAP=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2w_serial_$v.json 2>/dev/null
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2w_bench_$v.json 2>/dev/null
done
