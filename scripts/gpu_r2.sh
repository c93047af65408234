#!/bin/bash
# Round-2 GPU pass: parity at the large factors, the full GPU suite, config-5 sweep.
set -u
O=gpurun_out
mkdir -p $O
nproc > $O/r2_nproc.txt
timeout 900 python -m pytest tests/test_gpu_large.py -q -x --durations=0 > $O/r2_large.log 2>&1; echo "exit $?" >> $O/r2_large.log
timeout 1200 python -m pytest tests -m gpu -q > $O/r2_pytest.log 2>&1; echo "exit $?" >> $O/r2_pytest.log
timeout 600 python scripts/inverse_sweep.py --batch 2 --reps 3 > $O/r2_sweep.json 2> $O/r2_sweep.err; echo "exit $?" >> $O/r2_sweep.err
