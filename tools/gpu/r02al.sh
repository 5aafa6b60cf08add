#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02al; mkdir -p $O
timeout 2000 python -m pytest tests/test_reference_suite.py -m gpu -q -rf -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
