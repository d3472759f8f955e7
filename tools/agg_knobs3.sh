#!/bin/bash
# aggregation backward gather depth A/B (GFM_AGG_BWD_U / _MINB builds under
# paper_2406_12909_b200/_lib/<name>): in-step shapes (C3, C2) and the C5
# sweep at E = 16M
for lib in ${LIBS:-default u2m4 u4m3 u4m2 pf1 pf2}; do
  if [ $lib = default ]; then unset GFM_LIB_PATH; else export GFM_LIB_PATH=paper_2406_12909_b200/_lib/$lib/libgfm_b200.so; fi
  for c in c3 c2; do python tools/agg_time.py $c | sed "s/^/$lib /"; done
  python tools/agg_micro.py --e-list 16 --modes fused --reps 5 | sed "s/^/$lib /"
done
