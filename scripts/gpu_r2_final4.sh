#!/bin/bash
# Full pass of the current build: GPU suite, smoke, bench (default, with CPU baseline),
# reference arm, launch list and ncu captures of the two SYRK kernels.
set -u
O=gpurun_out
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs > $O/fin4_pytest.log 2>&1; echo "exit $?" >> $O/fin4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fin4_smoke.log 2>&1; echo "exit $?" >> $O/fin4_smoke.log
timeout 900 python bench.py > $O/fin4_bench.json 2> $O/fin4_bench.err; echo "exit $?" >> $O/fin4_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/fin4_ref.json 2> $O/fin4_ref.err; echo "exit $?" >> $O/fin4_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fin4_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-raw-e2e > $O/fin4_launches.log 2>&1
SPNGD_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:syrk_pair_kernel -c 1 -o $O/fin4_pair \
  python scripts/syrk_one.py 1 > $O/fin4_ncu_pair.log 2>&1
SPNGD_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3_kernel -c 1 -o $O/fin4_single \
  python scripts/syrk_one.py 1 > $O/fin4_ncu_single.log 2>&1
