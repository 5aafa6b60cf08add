#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
MLB_D2_BANDED=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_noband.json 2> $O/bench_noband.err; echo "bench noband rc=$?" >> $O/rc.txt
timeout 1200 python tools/shard_projection.py --worlds 8 --out $O/proj.json > $O/proj.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
MLB_SHARD_ONE_STREAM=1 timeout 1200 python tools/shard_projection.py --worlds 8 --out $O/proj_one.json > $O/proj_one.log 2>&1; echo "proj one rc=$?" >> $O/rc.txt
MLB_D2_BANDED=0 timeout 1200 python tools/shard_projection.py --worlds 8 --out $O/proj_noband.json > $O/proj_noband.log 2>&1; echo "proj noband rc=$?" >> $O/rc.txt
