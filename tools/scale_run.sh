#!/bin/bash
# Round-2 multi-GPU evidence on one box (run under gpurun --gpus 4): the
# NCCL tests (2 ranks: DP, sharded store, thread ranks) and the default bench line (C3 + nested C2 / ragged /
# C4) at N = 1, 2, 4 -> gpurun_out/scale/
mkdir -p gpurun_out/scale
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_sharded.py tests/test_gpu_thread_ranks.py -q > gpurun_out/scale/multi.log 2>&1
tail -3 gpurun_out/scale/multi.log
timeout 600 python bench.py --cpu-sample-s 4 > gpurun_out/scale/n1.json 2> gpurun_out/scale/n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $n > gpurun_out/scale/n$n.json 2> gpurun_out/scale/n$n.err
done
for n in 1 2 4; do
  python -c "import json; d=json.loads(open('gpurun_out/scale/n$n.json').read().strip().splitlines()[-1]); print($n, round(d['value']), round(d['ms_per_step'],3), d['load_balance']['lif'], d['c2']['value'], d['c4_egnn']['value'], d.get('sharded_store_fetch'))" || tail -5 gpurun_out/scale/n$n.err
done
