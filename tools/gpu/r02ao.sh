#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ao; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_configs.py tests/test_gpu_config5.py tests/test_gpu_segment.py -m gpu -q -rf -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
