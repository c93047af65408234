#!/bin/bash
# single-CTA factor problems chunked for their own launch (~4 waves)
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_large.py -q -x > $O/kc_tests.log 2>&1; echo "exit $?" >> $O/kc_tests.log
for v in 1 2 3; do
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 0 --no-raw-e2e > $O/kc_bench_$v.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"syrk_pair|gemm_tf32x3_kernel<3" --csv --log-file $O/kc_launches.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-raw-e2e > $O/kc_launches.log 2>&1
