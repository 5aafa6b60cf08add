#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ap; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1,2 --m 3,4 --sorted > $O/micro_sorted.log 2>&1; echo "micro sorted rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1 --m 4 > $O/micro_node.log 2>&1; echo "micro node rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --steps 30 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --steps 30 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
