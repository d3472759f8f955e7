mkdir -p gpurun_out/scale
for cfg in c2 c3; do
  timeout 400 python bench.py --config $cfg > gpurun_out/scale/${cfg}_n1.json 2> gpurun_out/scale/${cfg}_n1.err
  for n in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --config $cfg > gpurun_out/scale/${cfg}_n$n.json 2> gpurun_out/scale/${cfg}_n$n.err
  done
done
timeout 600 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/scale/multi.log 2>&1
tail -n1 gpurun_out/scale/*.json; tail -2 gpurun_out/scale/multi.log
