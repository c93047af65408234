#!/bin/bash
# Inverse-chain anatomy: one 4608^2 A (+ 512^2 G) factor, per-launch durations.
set -u
O=gpurun_out
mkdir -p $O
timeout 300 python scripts/inv_one.py 4 > $O/r2e_inv_one.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2e_inv_one_ncu.csv \
  python scripts/inv_one.py 2 > $O/r2e_ncu.log 2>&1; echo "ncu exit $?" >> $O/r2e_ncu.log
