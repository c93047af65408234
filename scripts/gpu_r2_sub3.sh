#!/bin/bash
# raw-input host steps: per-layer-group device im2col + SYRK as the raw inputs land (A/B)
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "host or raw" > $O/sub3_tests.log 2>&1; echo "exit $?" >> $O/sub3_tests.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "host" > $O/sub3_multi.log 2>&1; echo "exit $?" >> $O/sub3_multi.log
for v in 1 2; do
  timeout 600 python bench.py --steps 5 --e2e-steps 10 --no-cpu-baseline > $O/sub3_on_$v.json 2>/dev/null
  SPNGD_NO_SUBWAVES=1 timeout 600 python bench.py --steps 5 --e2e-steps 10 --no-cpu-baseline > $O/sub3_off_$v.json 2>/dev/null
done
