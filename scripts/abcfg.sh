#!/bin/bash
# grid table entries (SYSCD_GRID_CFG) on config 3
for c in ${CFGS:-3 4 5}; do
  SYSCD_GRID_CFG=$c timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt > gpurun_out/ab.log 2>&1
  echo -n "cfg $c: "; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/ab.log
done
