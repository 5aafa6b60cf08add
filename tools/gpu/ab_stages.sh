#!/bin/bash
# A/B of two in-tree builds (libmlb_a.so / libmlb_b.so) on the stage split of configs 4 and 2
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do for v in a b; do for c in 4 2; do
  echo "== $v cfg$c rep$rep" >> $O/stages.txt
  MLB_LIB_VARIANT=libmlb_$v.so timeout 300 python tools/stages_cfg.py --config $c >> $O/stages.txt 2>&1
done; done; done
