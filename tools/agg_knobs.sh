#!/bin/bash
# A/B of the aggregation-gather variants at the C3 / C2 in-step shapes.
mkdir -p gpurun_out
for c in c3 c2; do
  python tools/agg_time.py $c
  GFM_AGG_GC=1 python tools/agg_time.py $c
  GFM_AGG_CHUNK=32 python tools/agg_time.py $c
  GFM_AGG_CHUNK=64 python tools/agg_time.py $c
  GFM_AGG_CHUNK=128 python tools/agg_time.py $c
  GFM_AGG_GC=1 GFM_AGG_CHUNK=64 python tools/agg_time.py $c
  if [ -f paper_2406_12909_b200/_lib/var/libgfm_b200.so ]; then
    GFM_LIB_PATH=paper_2406_12909_b200/_lib/var/libgfm_b200.so python tools/agg_time.py $c | sed 's/^/VAR /'
    GFM_AGG_GC=1 GFM_LIB_PATH=paper_2406_12909_b200/_lib/var/libgfm_b200.so python tools/agg_time.py $c | sed 's/^/VAR /'
  fi
done
python - <<'PY'
import glob, numpy as np
for c in ("c3", "c2"):
    fs = sorted(glob.glob(f"gpurun_out/aggout_{c}_*.npy"))
    ref = np.load(fs[0])
    for f in fs[1:]:
        print(c, f, "bitwise equal" if np.array_equal(np.load(f), ref) else "DIFFERENT")
PY
