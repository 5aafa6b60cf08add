#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aq; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spread1_kernel|gather1_kernel" -s 2 -c 2 -o $O/d1_sorted python tools/stages_micro.py --d 1 --m 4 --sorted > $O/ncu_d1.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
