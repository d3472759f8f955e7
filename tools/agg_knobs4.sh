#!/bin/bash
# aggregation forward variants (GFM_AGG_FWD_MINB / _UF builds under
# paper_2406_12909_b200/_lib/<name>) at the in-step shapes
for lib in ${LIBS:-default fm3 fm6 fu2 fu8}; do
  if [ $lib = default ]; then unset GFM_LIB_PATH; else export GFM_LIB_PATH=paper_2406_12909_b200/_lib/$lib/libgfm_b200.so; fi
  for c in c3 c2; do python tools/agg_time.py $c | sed "s/^/$lib /"; done
done
