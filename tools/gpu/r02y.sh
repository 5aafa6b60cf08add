#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_fullsize.py -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1,2,3 --m 4 > $O/micro_node.log 2>&1; echo "micro rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1,2 --m 4 --sorted > $O/micro_sorted.log 2>&1; echo "micro sorted rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
