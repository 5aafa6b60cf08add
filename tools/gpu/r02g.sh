#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g; mkdir -p $O
for ns in 4 8 16 32 52; do MLB_PKSM_STREAMS=$ns timeout 300 python tools/bench_solver.py --config 3 > $O/solver_cfg3_s$ns.json 2>&1; done
