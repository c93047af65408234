#!/bin/bash
# 4 GPUs: NCCL K-invariance + ledger of every optimizer mode, then the 2-GPU bench line.
set -u
O=gpurun_out
mkdir -p $O
for m in default p2p wgrad host; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
    scripts/multi_gpu_check.py --mode $m > $O/mgpu4_$m.log 2>&1; echo "exit $?" >> $O/mgpu_$m.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/bench_4gpu.json 2> $O/bench_4gpu.err; echo "exit $?" >> $O/bench_4gpu.err
