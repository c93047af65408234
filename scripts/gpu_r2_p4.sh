#!/bin/bash
# world 4: multi-GPU oracle tests + bench at P = 2 and 4 on the current build
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -rs > $O/p4_multi.log 2>&1; echo "exit $?" >> $O/p4_multi.log
timeout 600 python bench.py --gpus 4 --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/p4_bench4.json 2>$O/p4_bench4.err
timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/p4_bench2.json 2>$O/p4_bench2.err
