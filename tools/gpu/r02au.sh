#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02au; mkdir -p $O
for c in 1 2 3 4; do
MLB_CELL_CTAS=$c timeout 900 python tools/shard_projection.py --worlds 8 --steps 10 --out $O/proj_c$c.json > $O/proj_c$c.log 2>&1; echo "c$c rc=$?" >> $O/rc.txt
done
