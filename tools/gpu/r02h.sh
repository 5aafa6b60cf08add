#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02h; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for rep in 1 2; do for v in a b; do for c in 3 2 4; do
  MLB_LIB_VARIANT=libmlb_$v.so timeout 300 python tools/bench_solver.py --config $c > $O/solver_cfg${c}_${v}_$rep.json 2>&1
done; done; done
