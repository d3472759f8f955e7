"""Print selected raw metrics of an .ncu-rep (all kernels in it).
python tools/ncu_raw.py rep.ncu-rep [regex ...]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pats = [re.compile(p) for p in (sys.argv[2:] or [
    r"^gpu__time_duration.sum$", r"^dram__bytes_(read|write)\.sum$", r"dram__throughput.avg.pct",
    r"^sm__pipe_tensor.*cycles_active.*pct", r"^sm__warps_active.avg.pct",
    r"^launch__registers_per_thread$", r"^launch__grid_size$", r"^launch__shared_mem_per_block_dynamic$", r"^lts__t_bytes.sum$", r"^sm__inst_issued.avg.pct_of_peak_sustained_active$",
    r"^smsp__inst_executed.sum$", r"^sm__warps_active.avg.pct", r"^l1tex__t_sector_hit_rate.pct$",
    r"^lts__t_sector_hit_rate.pct$", r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$",
    r"smsp__pcsamp_warps_issue_stalled_(long_scoreboard|barrier|wait|mio_throttle|lg_throttle|"
    r"short_scoreboard|math_pipe_throttle|not_selected|selected|membar|sleeping|no_instruction|"
    r"branch_resolving|dispatch_stall|drain|imc_miss|tex_throttle)$"])]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    name = vals[hdr.index("Kernel Name")][:80] if "Kernel Name" in hdr else "?"
    print("==", name)
    for i, h in enumerate(hdr):
        if any(p.search(h) for p in pats):
            print(f"   {h} = {vals[i]} {units[i]}")
