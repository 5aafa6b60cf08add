#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02o; mkdir -p $O
python tools/prof_micro.py 1e7 1 64 4 > $O/prof_micro.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread|gather_kernel|grid_sum" -c 6 -o $O/ncu_micro_d1 python tools/prof_micro.py 1e7 1 64 4 > $O/ncu_d1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread|gather_kernel|grid_sum" -c 6 -o $O/ncu_micro_d2 python tools/prof_micro.py 1e7 2 64 4 > $O/ncu_d2.log 2>&1
