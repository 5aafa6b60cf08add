#!/bin/bash
# A/B: the deterministic d=3 spread reduction (cell blocks -> brick merge -> R2) vs red.global.add into the grid
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_atomic; mkdir -p $O
for rep in 1 2; do for mode in 0 1; do for c in 2 4; do
  echo "== atomic=$mode cfg$c rep$rep" >> $O/stages.txt
  MLB_SPREAD_ATOMIC=$mode timeout 300 python tools/stages_cfg.py --config $c >> $O/stages.txt 2>&1
  MLB_SPREAD_ATOMIC=$mode timeout 300 python bench.py --workload cfg$c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg${c}_atomic$mode.json 2>> $O/bench.err
done; done; done
MLB_SPREAD_ATOMIC=1 timeout 600 python -m pytest tests/test_gpu_fastsum.py -m gpu -q > $O/pytest_atomic.log 2>&1
