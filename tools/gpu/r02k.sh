#!/bin/bash
# seq step graphs for 2-layer configs: solver A/B + GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02k; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for rep in 1 2; do for c in 2 4 3 1; do
  timeout 300 python tools/bench_solver.py --config $c > $O/solver_cfg${c}_$rep.json 2>&1
done; done
for c in 2 4; do MLB_SEQ_GRAPHS=0 timeout 300 python tools/bench_solver.py --config $c > $O/solver_cfg${c}_noseq.json 2>&1; done
