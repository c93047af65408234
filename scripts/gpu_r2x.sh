#!/bin/bash
# world 2: multi-GPU oracle tests + bench on the current build
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > $O/r2x_multi.log 2>&1; echo "exit $?" >> $O/r2x_multi.log
for v in 1 2; do
  timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/r2x_bench2_$v.json 2>$O/r2x_bench2_$v.err
done
