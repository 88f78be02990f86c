#!/bin/bash
# config-C epoch kernel time per environment setting:
#   scripts/env_variants.sh C "SYSCD_DENSE_CFG=8" "SYSCD_DENSE_CFG=9" ...
C=$1; shift
for v in "$@"; do
  echo "$v: $(env $v python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu --no-ttt 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["roofline"]["kernel_ms"],4), round(d["roofline"]["frac"],4), round(d["ms_per_step"],4), d["config"]["workers"])')"
done
