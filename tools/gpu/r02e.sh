#!/bin/bash
# round 2 pass e: batched CGS2 in the lockstep graphs; config-5 accuracy tests
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in 3 2 1; do
  timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2> $O/solver_cfg$c.err; echo "solver $c rc=$?" >> $O/rc.txt
done
MLB_PKSM_BATCHED_CGS=0 timeout 600 python tools/bench_solver.py --config 3 > $O/solver_cfg3_nobatch.json 2>&1
MLB_LOCKSTEP_MIN_T=1 timeout 600 python tools/bench_solver.py --config 2 > $O/solver_cfg2_lock1.json 2>&1
timeout 600 python tools/pksm_profile.py --config 3 > $O/pksm_profile_cfg3.txt 2>&1
