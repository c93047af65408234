#!/bin/bash
# 4 GPUs: multi-GPU parity tests (world 2 and 4) and the bench at N = 2 and 4.
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/r2l_gpus.txt
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -rs --durations=0 > $O/r2l_multi.log 2>&1; echo "exit $?" >> $O/r2l_multi.log
for N in 2 4; do
  timeout 600 python bench.py --gpus $N > $O/r2l_bench$N.json 2> $O/r2l_bench$N.err; echo "exit $?" >> $O/r2l_bench$N.err
done
