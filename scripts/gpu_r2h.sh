#!/bin/bash
# ncu of the 2-CTA SYRK and the single-CTA SYRK launch of the R50 step (full set), + launch list.
set -u
O=gpurun_out
mkdir -p $O
timeout 300 python scripts/syrk_one.py 2 > $O/r2h_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:syrk_pair_kernel -c 1 -o $O/r2h_pair \
  python scripts/syrk_one.py 1 > $O/r2h_ncu_pair.log 2>&1; echo "exit $?" >> $O/r2h_ncu_pair.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3_kernel -c 1 -o $O/r2h_single \
  python scripts/syrk_one.py 1 > $O/r2h_ncu_single.log 2>&1; echo "exit $?" >> $O/r2h_ncu_single.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2h_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-raw-e2e > $O/r2h_launches.log 2>&1; echo "exit $?" >> $O/r2h_launches.log
