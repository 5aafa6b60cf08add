#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ax; mkdir -p $O
timeout 600 python tools/stages_cfg.py --config 3 > $O/stages_cfg3.log 2>&1; echo "rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -c 60 -s 200 --csv --log-file $O/launches.csv python tools/bench_solver.py --config 3 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
