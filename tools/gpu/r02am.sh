#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02am; mkdir -p $O
timeout 1200 python tools/layer_projection.py --out $O/layer_proj.json > $O/layer_proj.log 2>&1; echo "rc=$?" >> $O/rc.txt
