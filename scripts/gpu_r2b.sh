#!/bin/bash
# Round-2 GPU pass on 2 GPUs: failure semantics, multi-GPU parity, bench N=1/2, reference arm.
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/r2b_gpus.txt
timeout 600 python -m pytest tests/test_gpu_step.py -q -x -k "failed or singular" > $O/r2b_fail.log 2>&1; echo "exit $?" >> $O/r2b_fail.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rs --durations=0 > $O/r2b_multi.log 2>&1; echo "exit $?" >> $O/r2b_multi.log
timeout 900 python bench.py > $O/r2b_bench1.json 2> $O/r2b_bench1.err; echo "exit $?" >> $O/r2b_bench1.err
timeout 600 python bench.py --gpus 2 --no-cpu-baseline > $O/r2b_bench2.json 2> $O/r2b_bench2.err; echo "exit $?" >> $O/r2b_bench2.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/r2b_ref.json 2> $O/r2b_ref.err; echo "exit $?" >> $O/r2b_ref.err
