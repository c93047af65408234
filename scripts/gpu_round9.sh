#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -x > $O/pytest_step9.log 2>&1; echo "pytest exit $?" >> $O/pytest_step9.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench9_1.json 2> $O/bench9_1.err; echo "exit $?" >> $O/bench9_1.err
for m in default p2p; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/multi_gpu_check.py --mode $m > $O/mgpu9_$m.log 2>&1; echo "exit $?" >> $O/mgpu9_$m.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 > $O/bench9_2.json 2> $O/bench9_2.err; echo "exit $?" >> $O/bench9_2.err
