#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ba; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 400 --csv --log-file $O/launches.csv python tools/pksm_hostprof.py > $O/ncu.log 2>&1; echo "rc=$?" >> $O/rc.txt
