#!/bin/bash
# DRAM bytes per launch of gfm_agg_fwd / gfm_agg_bwd on the bench workload
# (ncu --set full, one call each) -> gpurun_out/agg_traffic_<cfg>.json
cfg=${1:-c2}
mkdir -p gpurun_out
python tools/agg_probe.py --config $cfg --once > gpurun_out/aggt_plain.log 2>&1 || exit 1
# the setup step itself launches 3 k_agg_ kernels per layer (fwd, bwd prep,
# bwd gather): skip them
layers=$(python -c "import sys; sys.path.insert(0, '.'); from bench import CONFIGS; print(CONFIGS['$cfg']['layers'])")
ncu --set full --clock-control none -k regex:k_agg_ --launch-skip $((3 * layers)) -c 3 -o /tmp/aggt -f \
    python tools/agg_probe.py --config $cfg --once > gpurun_out/aggt_ncu.log 2>&1
ncu -i /tmp/aggt.ncu-rep --page raw --csv > gpurun_out/aggt_$cfg.raw.csv 2>/dev/null
python - "$cfg" <<'PY'
import csv, json, sys
cfg = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/aggt_{cfg}.raw.csv")))
h, u = rows[0], rows[1]
ks = []
for v in rows[2:]:
    d = dict(zip(h, v))
    def b(k):
        x = float(d[k]); unit = u[h.index(k)]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    ks.append((d["Kernel Name"][:60], b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
               float(d["gpu__time_duration.sum"])))
out = dict(config=cfg, kernels=[dict(name=n, dram_bytes=x, ns_or_us=t) for n, x, t in ks],
           agg_fwd_dram_bytes=ks[0][1], agg_bwd_dram_bytes=ks[1][1] + ks[2][1],
           how="ncu --set full --clock-control none (cache flush between kernels), "
               "tools/ncu_agg_traffic.sh; bwd = prep + gather launches")
json.dump(out, open(f"gpurun_out/agg_traffic_{cfg}.json", "w"), indent=1)
print(json.dumps(out))
PY
