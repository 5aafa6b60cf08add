#!/bin/bash
# end-of-round measurement: bench lines (ours + reference arm), launch list of the bench command,
# ncu --set full of the spread / gather kernels of the config-4 step, GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/final5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"spread|gather_kernel|lat_" -c 8 -o $O/ncu_full python tools/prof_step.py 1 cfg4 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in 1 2 3 4; do timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2>&1; done
timeout 1500 python tools/shard_projection.py --worlds 1 2 4 8 --out $O/shard_projection.json > $O/shard_projection.log 2>&1; echo "proj rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q -s -m gpu > $O/parity_configs.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
