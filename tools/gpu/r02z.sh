#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_config5.py tests/test_gpu_fullsize.py -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1,2 --m 4 > $O/micro_node.log 2>&1; echo "micro rc=$?" >> $O/rc.txt
timeout 600 python tools/stages_micro.py --d 1,2 --m 4 --sorted > $O/micro_sorted.log 2>&1; echo "micro sorted rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spread1_kernel|gather1_kernel" -s 2 -c 2 -o $O/d1_sorted python tools/stages_micro.py --d 1 --m 4 --sorted > $O/ncu_d1.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
