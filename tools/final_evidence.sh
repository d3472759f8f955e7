#!/bin/bash
# Round-end evidence on one box (gpurun --gpus 4): ncu full captures of the
# dominant kernels (single process), launch lists, then 1/2/4-GPU bench lines.
mkdir -p gpurun_out
./tools/ncu_one.sh c2 aggbwd "k_agg_bwd_vec" 0
./tools/ncu_one.sh c2 aggfwd "k_agg_fwd_vec" 0
./tools/ncu_one.sh c3 gemmfwd "128, gfm::tc::TcEpiBiasAct" 0
./tools/ncu_agg_traffic.sh c2
./tools/ncu_agg_traffic.sh c3
python tools/step_once.py --steps 2 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/step_once.py --steps 2 > gpurun_out/ncu.log 2>&1
python tools/step_once.py --config c3 --steps 2 > gpurun_out/c3plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/step_once.py --config c3 --steps 2 > gpurun_out/ncu_c3.log 2>&1
./tools/scale.sh c2
./tools/scale.sh c3
