#!/bin/bash
# parity smoke + bench (kernel-only) + optional ncu capture of the epoch kernel
timeout 300 python scripts/gpu_check.py > gpurun_out/check.log 2>&1; echo check_exit=$?
grep -E "^cfg" gpurun_out/check.log | cut -c1-150 | head -20
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-ttt ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step',round(d['ms_per_step'],4),'upd/s',round(d['value']),'kernel_ms',round(d['roofline']['kernel_ms'],4),'frac',round(d['roofline']['frac'],3), d['config']['workers'], d['clocks'])" || tail -20 gpurun_out/bench.log
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_epoch -s 4 -c 1 -o gpurun_out/$NCU python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-ttt ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
fi
