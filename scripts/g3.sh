#!/bin/bash
# config-3 grid kernel quick look: timeline + kernel-only bench
timeout 300 python scripts/timeline_grid.py 3 > gpurun_out/tl3.log 2>&1; head -12 gpurun_out/tl3.log
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt > gpurun_out/b3.log 2>&1
tail -1 gpurun_out/b3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'kernel', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'])" || tail -5 gpurun_out/b3.log
