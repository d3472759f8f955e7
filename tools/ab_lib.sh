#!/bin/bash
# A/B of the default in-tree library (A) against an alternative build (B,
# paper_2406_12909_b200/_lib/var/libgfm_b200.so, selected with GFM_LIB_PATH)
# on the bench workload(s): tools/ab_lib.sh [config ...] (default c2).
mkdir -p gpurun_out
V=paper_2406_12909_b200/_lib/var/libgfm_b200.so
CFGS=${@:-c2}
for c in $CFGS; do
for i in 1 2; do
python bench.py --config $c --steps 30 --warmup 5 --cpu-sample-s 0.5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c A', d['value'], d['e2e']['value'])" >> gpurun_out/ab.log
GFM_LIB_PATH=$V python bench.py --config $c --steps 30 --warmup 5 --cpu-sample-s 0.5 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c B', d['value'], d['e2e']['value'])" >> gpurun_out/ab.log
done
done
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
