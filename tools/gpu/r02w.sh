#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python tools/bench_solver.py --config 3 > $O/solver_cfg3.json 2> $O/solver_cfg3.err; echo "cfg3 rc=$?" >> $O/rc.txt
MLB_PKSM_DEVICE_COEFFS=0 timeout 600 python tools/bench_solver.py --config 3 > $O/solver_cfg3_host.json 2> $O/solver_cfg3_host.err; echo "cfg3 host rc=$?" >> $O/rc.txt
