#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ar; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_config5.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
