#!/bin/bash
# round 2 pass b: full GPU suite (sharded graph / solvers, config-4 full-size parity)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
