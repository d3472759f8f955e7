#!/bin/bash
# Round-2 profile refresh (run under gpurun, one GPU): launch lists + ncu
# summaries (tools/r02_profile.sh), DRAM traffic of the in-step aggregation
# kernels, the tf32 accumulation K-scan without / with the flush, and the C5
# sweep -> gpurun_out/
mkdir -p gpurun_out
tools/r02_profile.sh > gpurun_out/r02_profile.log 2>&1
for c in c3 c2; do tools/ncu_agg_traffic.sh $c > gpurun_out/aggt_$c.log 2>&1; done
{ echo "## GFM_TC_FLUSH_KB=0 (no flush)"; GFM_TC_FLUSH_KB=0 python tools/tf32_probe.py k;
  echo "## default (flush every 16 k-blocks)"; python tools/tf32_probe.py k; } > gpurun_out/tf32_k.txt 2>&1
timeout 2400 python tools/agg_micro.py --json gpurun_out/agg_micro.json > gpurun_out/agg_micro.txt 2>&1
tail -3 gpurun_out/agg_micro.txt
