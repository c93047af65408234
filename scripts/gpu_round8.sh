#!/bin/bash
# 1 GPU: full GPU suite, bench line, launch list of the current build.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu8.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu8.log
timeout 900 python bench.py > $O/bench8.json 2> $O/bench8.err; echo "bench exit $?" >> $O/bench8.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches8.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > $O/ncu_list8.log 2>&1; echo "ncu list exit $?" >> $O/ncu_list8.log
