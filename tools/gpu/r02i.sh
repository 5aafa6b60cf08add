#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/gpu/ab_stages.sh
O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_fullsize.py tests/test_gpu_config5.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
