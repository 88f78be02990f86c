#!/bin/bash
# config-2 epoch kernel time per variant library (partition-Gram experiments)
for v in "$@"; do
  if [ "$v" = base ]; then L=libsyscd_b200.so; else L=libsyscd_b200_$v.so; fi
  echo "$v: $(SYSCD_LIB_NAME=$L timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu --no-ttt 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["kernel"], round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4), round(d["ms_per_step"],4))')"
done
