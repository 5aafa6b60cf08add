#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02at; mkdir -p $O
MLB_DEBUG=1 timeout 900 python tools/shard_projection.py --worlds 8 --steps 5 > $O/proj.log 2>&1; echo "rc=$?" >> $O/rc.txt
