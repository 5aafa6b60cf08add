#!/bin/bash
# round 2 pass d: graph-captured lockstep PKSM -- GPU suite, solver A/B, reference suite via the shim
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=12 -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in 3 2 1 4; do
  timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg$c.json 2> $O/solver_cfg$c.err; echo "solver $c rc=$?" >> $O/rc.txt
  MLB_PKSM_GRAPHS=0 timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg${c}_nographs.json 2>&1; echo "solver $c nographs rc=$?" >> $O/rc.txt
done
for c in 2 4; do MLB_LOCKSTEP_MIN_T=1 timeout 600 python tools/bench_solver.py --config $c > $O/solver_cfg${c}_lock1.json 2>&1; echo "solver $c lock1 rc=$?" >> $O/rc.txt; done
timeout 600 python tools/pksm_profile.py --config 3 > $O/pksm_profile_cfg3.txt 2>&1
