#!/bin/bash
# N = 1, 2, 4 bench lines of one config on one box (run under gpurun --gpus 4)
cfg=${1:-c2}
mkdir -p gpurun_out
timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --cpu-sample-s 2 > gpurun_out/scale_${cfg}_1.log 2>&1
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --config $cfg --gpus $n --steps 20 --warmup 5 > gpurun_out/scale_${cfg}_$n.log 2>&1
done
for n in 1 2 4; do tail -1 gpurun_out/scale_${cfg}_$n.log | cut -c1-220; done
