#!/bin/bash
# config-3 epoch time per grid-table entry (SYSCD_GRID_CFG forces one)
for c in "$@"; do
  echo "cfg $c: $(SYSCD_GRID_CFG=$c python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4), d["config"]["workers"])')"
done
