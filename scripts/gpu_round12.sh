#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 > $O/bench12_4.json 2> $O/bench12_4.err; echo "exit $?" >> $O/bench12_4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
  scripts/stale_bench.py --batch 256 > $O/stale12_4.json 2> $O/stale12_4.err; echo "exit $?" >> $O/stale12_4.err
