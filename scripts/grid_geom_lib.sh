#!/bin/bash
# config-3 epoch time per (library variant, forced grid-table entry): scripts/grid_geom_lib.sh "lib1 lib2" "cfg1 cfg2"
for v in $1; do
  if [ "$v" = base ]; then L=libsyscd_b200.so; else L=libsyscd_b200_$v.so; fi
  for c in $2; do
    echo "$v cfg $c: $(SYSCD_LIB_NAME=$L SYSCD_GRID_CFG=$c timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4))')"
  done
done
