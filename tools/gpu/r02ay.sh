#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ay; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py -m gpu -q -rf -k "not side1000" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/bench_solver.py --config 3 > $O/solver_cfg3.json 2> $O/solver_cfg3.err; echo "cfg3 rc=$?" >> $O/rc.txt
MLB_PKSM_MULTI=0 timeout 600 python tools/bench_solver.py --config 3 > $O/solver_cfg3_nomulti.json 2> $O/solver_cfg3_nomulti.err; echo "cfg3 nomulti rc=$?" >> $O/rc.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --steps 30 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench cfg2 rc=$?" >> $O/rc.txt
