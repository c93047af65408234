#!/bin/bash
# 2 GPUs: NCCL K-invariance + ledger of every optimizer mode, then the 2-GPU bench line.
set -u
O=gpurun_out
mkdir -p $O
for m in default p2p p2p_sgd wgrad bn_full one_mc sgd host; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/multi_gpu_check.py --mode $m > $O/mgpu_$m.log 2>&1; echo "exit $?" >> $O/mgpu_$m.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 > $O/bench_2gpu.json 2> $O/bench_2gpu.err; echo "exit $?" >> $O/bench_2gpu.err
