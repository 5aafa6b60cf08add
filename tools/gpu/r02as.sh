#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02as; mkdir -p $O
for r in 1 2; do for v in libmlb_a.so libmlb_b.so libmlb_c.so; do
MLB_LIB_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_${v}_$r.json 2> $O/bench_${v}_$r.err; echo "bench $v $r rc=$?" >> $O/rc.txt
done; done
MLB_LIB_VARIANT=libmlb_b.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q > $O/pytest_b.log 2>&1; echo "pytest b rc=$?" >> $O/rc.txt
