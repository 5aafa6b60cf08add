#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02az; mkdir -p $O
timeout 600 python tools/pksm_hostprof.py > $O/hostprof.log 2>&1; echo "rc=$?" >> $O/rc.txt
