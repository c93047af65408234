#!/bin/bash
# config 4 with drifting captures (partial refreshes) after the re-plan upload ordering fix
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stale.py -q -x > $O/cfg3_stale_tests.log 2>&1; echo "exit $?" >> $O/cfg3_stale_tests.log
timeout 900 python scripts/stale_bench.py --batch 32 --steps 30 --drift 0.02 > $O/cfg3_stale_b32_drift.json 2>$O/cfg3_stale.err
timeout 1200 python scripts/stale_bench.py --batch 256 --steps 30 --drift 0.02 > $O/cfg3_stale_b256_drift.json 2>>$O/cfg3_stale.err
