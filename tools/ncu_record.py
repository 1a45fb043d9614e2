#!/usr/bin/env python
"""Record one `ncu --set full` capture: per-launch DRAM traffic into profiles/ncu_traffic.json
(the bench's roofline.traffic) and a reduced metric table into profiles/<tag>.txt.

usage: tools/ncu_record.py gpurun_out/<rep>.ncu-rep <cfgN> <tag>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, cfg, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].split("<")[0].replace("void ", "").strip()
        by = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            by += float(r[hdr.index(m)].replace(",", "")) * SCALE[units[hdr.index(m)]]
        traffic[short] = by
        lines.append(f"== {name}")
        for k in KEEP:
            if k in hdr:
                lines.append(f"  {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
    with open(os.path.join(ROOT, "profiles", f"{tag}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none capture {os.path.basename(rep)}\n")
        f.write("\n".join(lines) + "\n")
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d.setdefault(cfg, {}).update(traffic)
    d["source"] = d.get("source", {}) if isinstance(d.get("source"), dict) else {}
    for k in traffic:
        d["source"][f"{cfg}/{k}"] = f"profiles/{tag}.txt"
    with open(p, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
