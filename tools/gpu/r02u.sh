#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02u; mkdir -p $O
for cap in 1024 2048; do
MLB_CELL_CAP=$cap timeout 900 python tools/shard_projection.py --worlds 8 --out $O/proj_cap$cap.json > $O/proj_cap$cap.log 2>&1; echo "cap $cap rc=$?" >> $O/rc.txt
done
MLB_SPREAD_ATOMIC=1 timeout 900 python tools/shard_projection.py --worlds 8 --out $O/proj_atomic.json > $O/proj_atomic.log 2>&1; echo "atomic rc=$?" >> $O/rc.txt
MLB_WARP_SUBS=2 timeout 900 python tools/shard_projection.py --worlds 8 --out $O/proj_ws2.json > $O/proj_ws2.log 2>&1; echo "ws2 rc=$?" >> $O/rc.txt
