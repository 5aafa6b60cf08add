#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/gpu/ab_stages.sh
O=gpurun_out/r02l; mkdir -p $O
for v in a b; do MLB_LIB_VARIANT=libmlb_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$v.json 2>&1; done
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
MLB_D2_GTILE=1 timeout 900 python -m pytest tests/test_gpu_fastsum.py -m gpu -q -x -k "stages or tiny or large" > $O/pytest_gtile.log 2>&1; echo "pytest gtile rc=$?" >> $O/rc.txt
