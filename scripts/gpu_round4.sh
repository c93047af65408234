#!/bin/bash
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu4.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu4.log
bash scripts/kchunk_sweep.sh
