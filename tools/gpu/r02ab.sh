#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ab; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
for c in 2 4; do timeout 900 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2> $O/solver_cfg$c.err; echo "solver $c rc=$?" >> $O/rc.txt; done
