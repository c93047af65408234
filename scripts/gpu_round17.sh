#!/bin/bash
# Warp-per-row im2col: raw-input parity, the im2col launch under ncu, and the bench (e2e_raw_inputs).
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -k "raw" > $O/pytest17.log 2>&1; echo "pytest exit $?" >> $O/pytest17.log
timeout 600 python bench.py > $O/bench17.json 2> $O/bench17.err; echo "exit $?" >> $O/bench17.err
timeout 600 ncu --set full --clock-control none -k regex:im2col -c 1 -o $O/im2col17 -f python scripts/raw_step.py > $O/ncu_im2col17.log 2>&1
