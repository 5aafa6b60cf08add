#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fastsum.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded.json 2> $O/bench_sharded.err; echo "bench sharded rc=$?" >> $O/rc.txt
timeout 1200 python tools/shard_projection.py --out $O/shard_projection.json > $O/shard_projection.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
