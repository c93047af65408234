#!/bin/bash
# Final pass of the round: full GPU suite, smoke, 1-GPU bench, launch list.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_final.log 2>&1; echo "pytest exit $?" >> $O/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke exit $?" >> $O/smoke_final.log
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err; echo "exit $?" >> $O/bench_final.err
