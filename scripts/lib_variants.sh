#!/bin/bash
# config-C epoch kernel time per variant library: scripts/lib_variants.sh C name1 name2 ...
C=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then L=libsyscd_b200.so; else L=libsyscd_b200_$v.so; fi
  echo "$v: $(SYSCD_LIB_NAME=$L timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4), round(d["ms_per_step"],4))')"
done
