#!/bin/bash
# config 2 (ResNet-18 CIFAR) bench + reference arm; config 4 with drifting captures; stale GPU tests
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stale.py -q -x > $O/cfg_stale_tests.log 2>&1; echo "exit $?" >> $O/cfg_stale_tests.log
timeout 600 python bench.py --config resnet18 --steps 20 > $O/cfg_resnet18.json 2>$O/cfg_resnet18.err
timeout 600 python bench.py --config resnet18 --impl reference --steps 5 --warmup 1 > $O/cfg_resnet18_ref.json 2>$O/cfg_resnet18_ref.err
timeout 900 python scripts/stale_bench.py --batch 32 --steps 30 --drift 0.02 > $O/cfg_stale_b32_drift.json 2>$O/cfg_stale.err
timeout 1200 python scripts/stale_bench.py --batch 256 --steps 30 --drift 0.02 > $O/cfg_stale_b256_drift.json 2>>$O/cfg_stale.err
