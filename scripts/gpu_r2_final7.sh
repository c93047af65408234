#!/bin/bash
# last pass on a 4-GPU box: the whole -m gpu suite (world 1/2/4), smoke, bench at P = 1, 2, 4
set -u
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/fin7_pytest.log 2>&1; echo "exit $?" >> $O/fin7_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fin7_smoke.log 2>&1; echo "exit $?" >> $O/fin7_smoke.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/fin7_bench1.json 2>/dev/null
timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu-baseline --e2e-steps 3 --no-raw-e2e > $O/fin7_bench2.json 2>/dev/null
timeout 600 python bench.py --gpus 4 --steps 20 --no-cpu-baseline --e2e-steps 3 --no-raw-e2e > $O/fin7_bench4.json 2>/dev/null
