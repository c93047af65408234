#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q -k "step_host or overlapped or raw" > $O/pytest15.log 2>&1; echo "pytest exit $?" >> $O/pytest15.log
timeout 600 python bench.py > $O/bench15_1.json 2> $O/bench15_1.err; echo "exit $?" >> $O/bench15_1.err
