for cfg in "32 64" "64 128" "128 384"; do set -- $cfg; echo "NB=$1 CAP=$2"; GFM_AGG_TILE=1 GFM_AGG_TILE_NB=$1 GFM_AGG_TILE_CAP=$2 python tools/agg_probe.py --config c2 2>&1 | grep "^c2"; done
python tools/agg_probe.py --config c2 2>&1 | grep "^c2"
for cfg in "50 128" "100 256"; do set -- $cfg; echo "NB=$1 CAP=$2"; GFM_AGG_TILE=1 GFM_AGG_TILE_NB=$1 GFM_AGG_TILE_CAP=$2 python tools/agg_probe.py --config c3 2>&1 | grep "^c3"; done
python tools/agg_probe.py --config c3 2>&1 | grep "^c3"
