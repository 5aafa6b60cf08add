#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f; mkdir -p $O
bash tools/gpu/ab_stages.sh
timeout 900 python -m pytest tests/test_gpu_segment.py tests/test_gpu_solvers.py tests/test_cli.py -m gpu -q -rf -s > $O/pytest_seg.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for d in 2 3; do MLB_PKSM_DEPTH=$d timeout 300 python tools/bench_solver.py --config 3 > $O/solver_cfg3_depth$d.json 2>&1; done
