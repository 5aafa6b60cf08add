#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ag; mkdir -p $O
timeout 1200 python tools/shard_projection.py --worlds 8 --out $O/proj.json > $O/proj.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
