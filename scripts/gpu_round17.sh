#!/bin/bash
# Warp-per-row im2col and 32-bit unpack_damp: full GPU suite, the bench (incl. e2e_raw_inputs), both kernels under ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest17.log 2>&1; echo "pytest exit $?" >> $O/pytest17.log
timeout 600 python bench.py > $O/bench17.json 2> $O/bench17.err; echo "exit $?" >> $O/bench17.err
timeout 600 ncu --set full --clock-control none -k regex:im2col -c 1 -o $O/im2col17 -f python scripts/raw_step.py > $O/ncu_im2col17.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:unpack_damp -c 1 -o $O/unpack17 -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_unpack17.log 2>&1
