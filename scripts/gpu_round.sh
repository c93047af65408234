#!/bin/bash
# One gpurun pass: GPU parity tests, 1-GPU bench line, ncu launch list and a
# full capture of the factor SYRK launch.  Outputs under gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench exit $?" >> $O/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $O/ncu_list.log 2>&1; echo "ncu list exit $?" >> $O/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -c 1 \
  -o $O/factor_gemm -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $O/ncu_full.log 2>&1; echo "ncu full exit $?" >> $O/ncu_full.log
