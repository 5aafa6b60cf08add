#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bb; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --steps 30 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
