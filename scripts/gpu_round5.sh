#!/bin/bash
# Config 4 at its own batch (256/GPU) and the config-5 inverse sweep, 1 GPU.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python scripts/stale_bench.py --batch 256 > $O/stale_b256_1gpu.json 2> $O/stale_b256_1gpu.err; echo "exit $?" >> $O/stale_b256_1gpu.err
timeout 900 python scripts/inverse_sweep.py > $O/inverse_sweep.json 2> $O/inverse_sweep.err; echo "exit $?" >> $O/inverse_sweep.err
