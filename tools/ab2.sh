#!/bin/bash
# A/B of the in-tree library (A) against paper_2406_12909_b200/_lib/var (B):
# tools/ab2.sh [config ...]; prints value and ms_per_step per run.
mkdir -p gpurun_out
V=paper_2406_12909_b200/_lib/var/libgfm_b200.so
for c in ${@:-c2}; do
for i in 1 2; do
for arm in A B; do
if [ $arm = B ]; then export GFM_LIB_PATH=$V; else unset GFM_LIB_PATH; fi
python bench.py --config $c --steps 30 --warmup 5 --cpu-sample-s 0.5 --no-nested 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $arm', round(d['value']), round(d['ms_per_step'], 4), d['clocks']['sm_mhz'])"
done; done; done
