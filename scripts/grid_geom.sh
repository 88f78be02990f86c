#!/bin/bash
# config-3 epoch time per forced grid-table entry, with and without spreading d evenly over the CTAs
for c in "$@"; do
  for sp in ${SPREADS:-""}; do
    echo "cfg $c spread=${sp:-0}: $(SYSCD_GRID_SPREAD=$sp SYSCD_GRID_CFG=$c timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4))')"
  done
done
