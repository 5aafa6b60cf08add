#!/bin/bash
# round 2, first GPU pass: smoke, GPU tests, config-4 bench, launch list + traffic, ncu full on the top kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:randomly > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench cfg4 rc=$?" >> $O/rc.txt
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ncu_cfg4_step.csv python tools/prof_step.py 2 cfg4 > $O/ncu_cfg4_step.log 2>&1; echo "ncu step rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread|gather" -c 4 -o $O/ncu_cfg4_full python tools/prof_step.py 1 cfg4 > $O/ncu_cfg4_full.log 2>&1; echo "ncu full rc=$?" >> $O/rc.txt
