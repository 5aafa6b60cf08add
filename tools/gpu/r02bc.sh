#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bc; mkdir -p $O
for sp in 256 512 1024; do
MLB_SEG_POINTS=$sp timeout 600 python tools/bench_solver.py --config 3 > $O/solver_sp$sp.json 2> $O/solver_sp$sp.err; echo "sp$sp rc=$?" >> $O/rc.txt
done
