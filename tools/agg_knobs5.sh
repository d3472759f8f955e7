#!/bin/bash
# deep gather batch (GFM_AGG_BWD_U_DEEP builds) on the C5 random sweep at E = 16M
for lib in ${LIBS:-default ud3 ud4}; do
  if [ $lib = default ]; then unset GFM_LIB_PATH; else export GFM_LIB_PATH=paper_2406_12909_b200/_lib/$lib/libgfm_b200.so; fi
  python tools/agg_micro.py --e-list 16 --modes fused --reps 5 --patterns random | sed "s/^/$lib /"
done
