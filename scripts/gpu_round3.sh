#!/bin/bash
# Full GPU suite + 1-GPU bench (e2e through spngd_opt_step_host, raw-input e2e).
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu3.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu3.log
timeout 900 python bench.py > $O/bench3.json 2> $O/bench3.err; echo "bench exit $?" >> $O/bench3.err
