#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02p; mkdir -p $O
for v in a b; do for so in "" "--sorted"; do
  echo "== $v $so" >> $O/micro.txt
  MLB_LIB_VARIANT=libmlb_$v.so timeout 600 python tools/stages_micro.py --d 1,2 --m 4 $so >> $O/micro.txt 2>&1
done; done
MLB_LIB_VARIANT=libmlb_b.so timeout 900 python -m pytest tests/test_gpu_fastsum.py tests/test_gpu_config5.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
