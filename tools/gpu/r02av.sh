#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02av; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --steps 30 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --steps 30 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
timeout 1200 python tools/shard_projection.py --worlds 2 4 8 --out $O/proj.json > $O/proj.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
