#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02r; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=8 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded.json 2> $O/bench_sharded.err; echo "bench sharded rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
