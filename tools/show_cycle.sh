#!/bin/bash
cat gpurun_out/probe.log | grep -v "^shape" | awk '{print $1,$2,$3,$4,$5,$6,$8}'
grep -E "FAILED|passed|failed|Error" gpurun_out/gpu_tests.log | head -8
python -c "
import json;l=open('gpurun_out/bench.log').read().strip().splitlines()[-1]
d=json.loads(l);print('bench: %.0f graphs/s  %.3f ms/step  e2e %.0f  agg roofline %.2f'%(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac']))" 2>/dev/null || tail -3 gpurun_out/bench.log
python tools/ncu_summary.py gpurun_out/launches.csv 2 2>/dev/null | head -${1:-16}
