#!/bin/bash
# host-input steps: last wave's SYRK by layer groups as their captures land (A/B vs one launch)
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "host or raw" > $O/sub_tests.log 2>&1; echo "exit $?" >> $O/sub_tests.log
for v in 1 2; do
  timeout 600 python bench.py --steps 5 --e2e-steps 10 --no-cpu-baseline --no-raw-e2e > $O/sub_on_$v.json 2>/dev/null
  SPNGD_NO_SUBWAVES=1 timeout 600 python bench.py --steps 5 --e2e-steps 10 --no-cpu-baseline --no-raw-e2e > $O/sub_off_$v.json 2>/dev/null
done
