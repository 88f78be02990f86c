#!/bin/bash
# Every BASELINE config through both bench arms (driver defaults: 20 steps, 5 warm-up).
# Usage (GPU box): bash scripts/all_configs.sh <round-tag>
R=${1:-r2}
for c in 3 2 1 0 4; do
  timeout 900 python bench.py --config $c > gpurun_out/${R}_bench_cfg$c.json 2> gpurun_out/${R}_bench_cfg$c.err
  echo "cfg $c ours rc=$?"
  timeout 900 python bench.py --config $c --impl reference > gpurun_out/${R}_ref_cfg$c.json 2> gpurun_out/${R}_ref_cfg$c.err
  echo "cfg $c reference rc=$?"
done
