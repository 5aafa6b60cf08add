#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02n; mkdir -p $O
timeout 600 python tools/stages_micro.py --d 1,2 --m 3,4,6 > $O/stages_micro.txt 2>&1
timeout 600 python tools/stages_micro.py --d 3 --m 4 >> $O/stages_micro.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
