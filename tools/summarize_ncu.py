#!/usr/bin/env python
"""Summarise ncu output from gpurun_out/ into profiles/<tag>_summary.md (+ ncu_traffic.json).

Inputs (written by tools/profile_all.sh <tag>):
  <tag>_launches_cfgN.csv  launch lists (gpu__time_duration.sum, cold + serialised)
  <tag>_full_<name>_raw.csv one `ncu --set full` capture per dominant kernel
The raw metric tables are copied to profiles/ in reduced form (selected metrics only).
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "TC pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_sb"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def read_launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')]
    if not start:
        return None
    rows = list(csv.DictReader(lines[start[0]:]))
    agg = collections.OrderedDict()
    for r in rows:
        agg.setdefault(r["Kernel Name"], []).append(float(r["Metric Value"]) * 1e-3)  # ns -> us
    return agg


def read_raw(path):
    r = list(csv.reader(open(path)))
    if len(r) < 3:
        return None
    hdr, units, vals = r[0], r[1], r[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def to_si(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(u, 1.0)


def main(tag):
    out = [f"# ncu summary — {tag}", "",
           "Produced by `tools/profile_all.sh {0}` under gpurun on one B200, summarised by "
           "`tools/summarize_ncu.py {0}`. Launch lists are `gpu__time_duration.sum` with "
           "`--clock-control none` (cold-cache, serialised: compare shares, not absolutes). "
           "Full captures are `ncu --set full --clock-control none --import-source on`, one "
           "launch each.".format(tag), ""]
    out += ["## Launch lists", ""]
    for cfg in (2, 3, 4, 5):
        p = os.path.join(SRC, f"{tag}_launches_cfg{cfg}.csv")
        if not os.path.exists(p):
            continue
        agg = read_launches(p)
        if not agg:
            continue
        tot = sum(sum(v) for v in agg.values())
        out += [f"### cfg{cfg}", "", "| kernel | launches | mean µs | share |", "|---|---|---|---|"]
        for k, v in agg.items():
            out.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.2f} |")
        out.append("")
        with open(os.path.join(DST, f"{tag}_launches_cfg{cfg}.csv"), "w") as f:
            f.write("kernel,duration_us\n")
            for k, v in agg.items():
                for x in v:
                    f.write(f"\"{k}\",{x:.3f}\n")
    out += ["## Full captures", ""]
    traffic = {}
    tp = os.path.join(DST, "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for fn in sorted(os.listdir(SRC)):
        if not (fn.startswith(f"{tag}_full_") and fn.endswith("_raw.csv")):
            continue
        name = fn[len(f"{tag}_full_"):-len("_raw.csv")]
        got = read_raw(os.path.join(SRC, fn))
        if not got:
            continue
        d, kname = got
        out += [f"### {name}: `{kname[:80]}`", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in d:
                v, u = d[m]
                out.append(f"| {label} (`{m}`) | {v} {u} |")
        rd = to_si(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wr = to_si(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        if rd is not None and wr is not None:
            cfg = name.split("_")[0]
            kbase = kname.split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
            traffic.setdefault(cfg, {})[kbase] = rd + wr
        out.append("")
        sel = {m: d[m] for m, _ in METRICS if m in d}
        with open(os.path.join(DST, f"{tag}_full_{name}.json"), "w") as f:
            json.dump({"kernel": kname, "metrics": sel}, f, indent=1)
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one "
                        "ncu --set full capture (profiles/<tag>_summary.md)")
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    with open(os.path.join(DST, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
