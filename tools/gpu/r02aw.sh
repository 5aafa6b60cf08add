#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aw; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py -m gpu -q -rf -k "not side1000" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in 3 2; do timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2> $O/solver_cfg$c.err; echo "cfg$c rc=$?" >> $O/rc.txt; done
