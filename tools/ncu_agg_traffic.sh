#!/bin/bash
# DRAM bytes per launch of gfm_agg_fwd / gfm_agg_bwd (prep + gather) at a
# bench config's in-step shape (tools/agg_time.py: uint8 argmax as in the
# step), ncu --set full (cache flush between kernels)
#   -> gpurun_out/agg_traffic_<cfg>.json (bench.py's roofline.traffic)
cfg=${1:-c3}
mkdir -p gpurun_out
python tools/agg_time.py $cfg > gpurun_out/aggt_plain_$cfg.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:k_agg_fwd -c 1 -o /tmp/aggt_f -f \
    python tools/agg_time.py $cfg > gpurun_out/aggt_ncu_f.log 2>&1
ncu --set full --clock-control none -k regex:k_agg_bwd -c 2 -o /tmp/aggt_b -f \
    python tools/agg_time.py $cfg > gpurun_out/aggt_ncu_b.log 2>&1
ncu -i /tmp/aggt_f.ncu-rep --page raw --csv > gpurun_out/aggt_f_$cfg.raw.csv 2>/dev/null
ncu -i /tmp/aggt_b.ncu-rep --page raw --csv > gpurun_out/aggt_b_$cfg.raw.csv 2>/dev/null
python - "$cfg" <<'PY'
import csv, json, sys
cfg = sys.argv[1]
ks = []
for part in ("f", "b"):
    rows = list(csv.reader(open(f"gpurun_out/aggt_{part}_{cfg}.raw.csv")))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        def b(k):
            x = float(d[k]); unit = u[h.index(k)]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        ks.append((d["Kernel Name"][:70], b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
                   float(d["gpu__time_duration.sum"]), u[h.index("gpu__time_duration.sum")]))
out = dict(config=cfg, flags=2, kernels=[dict(name=n, dram_bytes=x, time=t, time_unit=tu)
                                         for n, x, t, tu in ks],
           agg_fwd_dram_bytes=ks[0][1], agg_bwd_dram_bytes=sum(k[1] for k in ks[1:]),
           source="profiles/r02_agg_traffic_%s.json (tools/ncu_agg_traffic.sh)" % cfg,
           how="ncu --set full --clock-control none (cache flush between kernels) on "
               "tools/agg_time.py; bwd = prep + gather launches; uint8 argmax as in the step")
json.dump(out, open(f"gpurun_out/agg_traffic_{cfg}.json", "w"), indent=1)
print(json.dumps(out))
PY
