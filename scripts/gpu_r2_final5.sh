#!/bin/bash
# last full pass: GPU suite, smoke, default bench (CPU baseline, e2e), reference arm
set -u
O=gpurun_out
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs > $O/fin5_pytest.log 2>&1; echo "exit $?" >> $O/fin5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fin5_smoke.log 2>&1; echo "exit $?" >> $O/fin5_smoke.log
timeout 900 python bench.py > $O/fin5_bench.json 2> $O/fin5_bench.err; echo "exit $?" >> $O/fin5_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/fin5_ref.json 2> $O/fin5_ref.err; echo "exit $?" >> $O/fin5_ref.err
