#!/bin/bash
# A/B of the config-3 epoch kernel: SYSCD_LIB_NAME=<variant .so> vs the current build
for lib in ${AB_LIBS:-libsyscd_b200_orig.so libsyscd_b200.so libsyscd_b200_orig.so libsyscd_b200.so}; do
  SYSCD_LIB_NAME=$lib timeout 300 python bench.py --config ${CFG:-3} --steps 5 --warmup 3 --no-e2e --no-cpu --no-ttt > gpurun_out/ab.log 2>&1
  echo -n "$lib: "; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'kernel', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/ab.log
done
