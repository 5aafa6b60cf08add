#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/gpu/ab_atomic.sh
O=gpurun_out/r02j; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
