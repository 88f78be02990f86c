#!/bin/bash
# Second-session refresh (GPU box): both bench arms for every config, then one
# --set full capture of the sparse epoch kernel.
bash scripts/all_configs.sh r2b
B4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt"
$B4 > gpurun_out/plain4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sparse_epoch -s 1 -c 1 -o gpurun_out/r2b_cfg4_sparse $B4 > /dev/null 2>&1
echo cfg4ncu=$?
