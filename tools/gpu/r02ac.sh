#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ac; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
