#!/bin/bash
# round 2 pass c: device bind -- GPU suite, config-4 bench, solver pipelines (config 1-4)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench rc=$?" >> $O/rc.txt
for c in 1 2 3 4; do timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2> $O/solver_cfg$c.err; echo "solver $c rc=$?" >> $O/rc.txt; done
