#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3; do
  timeout 300 python tools/agg_probe.py --config $c
  GFM_AGG_TILE=1 timeout 300 python tools/agg_probe.py --config $c
done > gpurun_out/agg_ab.log 2>&1
cat gpurun_out/agg_ab.log | grep -v Warn
