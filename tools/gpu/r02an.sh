#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02an; mkdir -p $O
for combo in "8 4" "2 1" "4 2" "2 4" "8 1" "1 1"; do
set -- $combo
MLB_GATHER_WARPS_D2=$1 MLB_BAND_WARPS=$2 timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_g$1_b$2.json 2> $O/bench_g$1_b$2.err; echo "g$1 b$2 rc=$?" >> $O/rc.txt
done
