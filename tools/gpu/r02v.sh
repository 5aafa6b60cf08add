#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_bench_cli.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded.json 2> $O/bench_sharded.err; echo "bench sharded rc=$?" >> $O/rc.txt
MLB_SHARD_JOINED=1 timeout 900 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded_joined.json 2> $O/bench_sharded_joined.err; echo "bench sharded joined rc=$?" >> $O/rc.txt
timeout 1200 python tools/shard_projection.py --worlds 2 4 8 --out $O/proj.json > $O/proj.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
MLB_SHARD_JOINED=1 timeout 1200 python tools/shard_projection.py --worlds 8 --out $O/proj_joined.json > $O/proj_joined.log 2>&1; echo "proj joined rc=$?" >> $O/rc.txt
