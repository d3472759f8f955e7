#!/bin/bash
# aggregation variants: compile-time (GFM_AGG_BWD_U / _MINB builds under
# paper_2406_12909_b200/_lib/<name>) and the fused bwd-data + prep epilogue
for lib in default u4 u1 minb3 minb8; do
  if [ $lib = default ]; then unset GFM_LIB_PATH; else export GFM_LIB_PATH=paper_2406_12909_b200/_lib/$lib/libgfm_b200.so; fi
  for c in c3 c2; do python tools/agg_time.py $c | sed "s/^/$lib /"; done
done
unset GFM_LIB_PATH
for fp in 0 1; do
  for c in c3 c2; do
    GFM_FUSED_PREP=$fp python bench.py --config $c --steps 30 --warmup 5 --cpu-sample-s 0.5 --no-nested 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FUSED_PREP=$fp $c', round(d['value']), round(d['ms_per_step'], 4))"
  done
done
