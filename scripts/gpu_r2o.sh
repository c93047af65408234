#!/bin/bash
# DRAM bytes of the factor-SYRK launches with explicit vs implicit im2col.
set -u
O=gpurun_out
mkdir -p $O
for M in explicit implicit; do
  F=""; [ $M = implicit ] && F="--implicit"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"syrk_pair_kernel|gemm_tf32x3_kernel|im2col_kernel|repack_kernel" --csv --log-file $O/r2o_$M.csv \
    python scripts/raw_step.py $F > $O/r2o_$M.log 2>&1
done
