#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ah; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_bench_cli.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded.json 2> $O/bench_sharded.err; echo "bench sharded rc=$?" >> $O/rc.txt
timeout 900 python bench.py --sharded --no-cpu-baseline --no-cuda-graph > $O/bench_sharded_eager.json 2> $O/bench_sharded_eager.err; echo "bench sharded eager rc=$?" >> $O/rc.txt
