#!/bin/bash
# ncu of the factor SYRK's 2-CTA launch, ungraphed (kernel replay of a graph-captured PDL launch hung)
set -u
O=gpurun_out
mkdir -p $O
SPNGD_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:syrk_pair_kernel -c 1 -o $O/fin2_pair \
  python scripts/syrk_one.py 1 > $O/fin2_ncu_pair.log 2>&1
