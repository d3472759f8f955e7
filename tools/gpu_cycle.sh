#!/bin/bash
# Standard GPU check: probe, tests, bench, launch list (run under gpurun).
mkdir -p gpurun_out
timeout 300 python tools/gemm_probe.py > gpurun_out/probe.log 2>&1
timeout 400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-sample-s 2 > gpurun_out/bench.log 2>&1
python tools/step_once.py --steps 2 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/step_once.py --steps 2 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/gpu_tests.log
