#!/bin/bash
# Round profiles (GPU box): the launch list of the default bench command and
# one --set full capture per epoch kernel.  Usage: bash scripts/profile_round.sh r2
R=${1:-r2}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-ttt"
$B > gpurun_out/plain_default.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_cfg3.csv $B > /dev/null 2>&1
echo launches=$?
B3="python bench.py --config 3 --steps 1 --warmup 2 --no-e2e --no-cpu --no-ttt"
$B3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grid_epoch -s 2 -c 1 -o gpurun_out/${R}_cfg3_grid $B3 > /dev/null 2>&1
echo cfg3=$?
B2="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-ttt"
$B2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_epoch -s 4 -c 1 -o gpurun_out/${R}_cfg2_dense $B2 > /dev/null 2>&1
echo cfg2=$?
B4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt"
$B4 > gpurun_out/plain4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sparse_epoch -s 1 -c 1 -o gpurun_out/${R}_cfg4_sparse $B4 > /dev/null 2>&1
echo cfg4=$?
