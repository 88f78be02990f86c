#!/bin/bash
# The N>1 bench path on ONE GPU: two ranks over gloo (host-staged collectives,
# no kernel waits on another rank).  Exercises shard-local generation, the
# per-round dv all-reduce, the alpha all-gather and both arms' rank handling;
# the numbers are not benchmarks.  Usage (GPU box): bash scripts/multi_rank_smoke.sh
export SYSCD_BENCH_BACKEND=gloo
for c in 3 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + c)) bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-cpu \
    > gpurun_out/mr_cfg$c.json 2> gpurun_out/mr_cfg$c.err
  echo "cfg $c ours N=2 rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29510 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 \
  > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref N=2 rc=$?"
