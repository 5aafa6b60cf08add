#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ae; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_configs.py -m gpu -q -rf -s -k side1000 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
