#!/bin/bash
# same-box A/B: inverse-recursion GEMMs on the 2-CTA kernel vs the 128-row kernel.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_large.py -q -x > $O/r2r_tests.log 2>&1; echo "exit $?" >> $O/r2r_tests.log
for v in 1 2; do
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2r_bench_pair$v.json 2>/dev/null
SPNGD_NO_PAIR_INV=1 timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/r2r_bench_nopairinv$v.json 2>/dev/null
done
timeout 900 python scripts/inverse_sweep.py > $O/r2r_sweep_pair.json 2>$O/r2r_sweep.err
SPNGD_NO_PAIR_INV=1 timeout 900 python scripts/inverse_sweep.py > $O/r2r_sweep_nopairinv.json 2>>$O/r2r_sweep.err
