#!/bin/bash
# bucketed vs single allreduce at N GPUs (C3, run under gpurun --gpus N)
n=${1:-4}
for mb in 4 0 16; do for i in 1 2; do
GFM_BUCKET_MB=$mb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-nested 2>/dev/null | tail -n1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bucket_mb=$mb', $n, round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
done; done
