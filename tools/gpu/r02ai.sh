#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fastsum.py -m gpu -q -rf -k "banded or stages" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do for v in libmlb_a.so libmlb_b.so; do
MLB_LIB_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_${v}_$r.json 2> $O/bench_${v}_$r.err; echo "bench $v $r rc=$?" >> $O/rc.txt
done; done
