#!/bin/bash
# world 2/4: late precondition stages before the update inside the schedule
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -rs > $O/p4b_multi.log 2>&1; echo "exit $?" >> $O/p4b_multi.log
for v in 1 2; do
  timeout 600 python bench.py --gpus 4 --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/p4b_bench4_$v.json 2>/dev/null
  timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/p4b_bench2_$v.json 2>/dev/null
done
