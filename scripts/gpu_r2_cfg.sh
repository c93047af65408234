#!/bin/bash
# configs 1/2 (MLP, ResNet-18 CIFAR) bench lines + reference arms; config 4 with fixed and drifting captures
set -u
O=gpurun_out
mkdir -p $O
for c in mlp resnet18; do
  timeout 600 python bench.py --config $c --steps 20 > $O/cfg_${c}.json 2>$O/cfg_${c}.err
  timeout 600 python bench.py --config $c --impl reference --steps 5 --warmup 1 > $O/cfg_${c}_ref.json 2>$O/cfg_${c}_ref.err
done
timeout 900 python scripts/stale_bench.py --batch 32 --steps 30 > $O/cfg_stale_b32_fixed.json 2>$O/cfg_stale.err
timeout 900 python scripts/stale_bench.py --batch 32 --steps 30 --drift 0.02 > $O/cfg_stale_b32_drift.json 2>>$O/cfg_stale.err
timeout 1200 python scripts/stale_bench.py --batch 256 --steps 30 --drift 0.02 > $O/cfg_stale_b256_drift.json 2>>$O/cfg_stale.err
timeout 1200 python scripts/stale_bench.py --batch 256 --steps 30 > $O/cfg_stale_b256_fixed.json 2>>$O/cfg_stale.err
