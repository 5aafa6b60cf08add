#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02q; mkdir -p $O
for sp in default 2048 1024 512; do
  if [ "$sp" = "default" ]; then unset MLB_SEG_POINTS; else export MLB_SEG_POINTS=$sp; fi
  echo "== seg $sp" >> $O/micro.txt
  timeout 600 python tools/stages_micro.py --d 1,2 --m 4 >> $O/micro.txt 2>&1
  echo "== seg $sp cfg4" >> $O/micro.txt
  timeout 600 python tools/stages_cfg.py --config 4 >> $O/micro.txt 2>&1
done
