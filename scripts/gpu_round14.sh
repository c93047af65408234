#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q > $O/pytest14.log 2>&1; echo "pytest exit $?" >> $O/pytest14.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench14_1.json 2> $O/bench14_1.err; echo "exit $?" >> $O/bench14_1.err
for m in p2p bn_full; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/multi_gpu_check.py --mode $m > $O/mgpu14_$m.log 2>&1; echo "exit $?" >> $O/mgpu14_$m.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 > $O/bench14_2.json 2> $O/bench14_2.err; echo "exit $?" >> $O/bench14_2.err
