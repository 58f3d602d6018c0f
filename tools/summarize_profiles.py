"""Turn ncu reports / launch lists from gpurun_out/ into committed summaries.

    python tools/summarize_profiles.py --tag round1 \
        --rep gpurun_out/prof_bfs.ncu-rep [--rep ...] --launches gpurun_out/launches_bfs.csv [...]

Writes profiles/<tag>_ncu.md (per-kernel metrics + stall mix), appends
launch-list shares to profiles/<tag>_launches.md and updates
profiles/ncu_traffic.json (dram bytes per launch of each kernel, read by
bench.py for the roofline "traffic" field).
"""
import argparse
import csv
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = OrderedDict([
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 rd sect"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sect"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
    ("launch__registers_per_thread", "regs"),
])
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def val(hdr, units, row, name):
    if name not in hdr:
        return None
    i = hdr.index(name)
    s = row[i].replace(",", "")
    try:
        x = float(s)
    except ValueError:
        return None
    return x * UNIT.get(units[i], 1.0)


def stalls(hdr, row):
    items = []
    for h, x in zip(hdr, row):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                items.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", ""))))
            except ValueError:
                pass
    tot = sum(x for _, x in items) or 1.0
    items.sort(key=lambda t: -t[1])
    return ", ".join(f"{k} {x / tot:.0%}" for k, x in items[:4])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    traffic = {}  # kernels captured now replace their old entries
    lines = [f"# ncu --set full summaries ({args.tag}) {args.title}", "",
             "Per launch; `ncu --set full --clock-control none` (serialised, cold caches).", ""]
    for rep in args.rep:
        hdr, units, rows = raw(rep)
        ki = hdr.index("Kernel Name")
        lines.append(f"## {os.path.basename(rep)}")
        lines.append("")
        lines.append("| kernel | " + " | ".join(METRICS.values()) + " | top stalls |")
        lines.append("|" + "---|" * (len(METRICS) + 2))
        for r in rows:
            name = r[ki].split("(")[0].replace("void ", "").replace("gb::", "")
            cells = []
            for m in METRICS:
                v = val(hdr, units, r, m)
                if v is None:
                    cells.append("-")
                elif m.startswith("gpu__time"):
                    cells.append(f"{v * 1e6:.1f} us")
                elif m.startswith("dram__bytes"):
                    cells.append(f"{v / 1e6:.1f} MB")
                elif "sectors" in m:
                    cells.append(f"{v / 1e6:.1f} M")
                else:
                    cells.append(f"{v:.1f}")
            lines.append(f"| {name} | " + " | ".join(cells) + f" | {stalls(hdr, r)} |")
            rd = val(hdr, units, r, "dram__bytes_read.sum") or 0.0
            wr = val(hdr, units, r, "dram__bytes_write.sum") or 0.0
            key = name.split("<")[0]
            prev = traffic.get(key)
            # keep the largest launch per kernel (the dominant one a bench line cites)
            if prev is None or rd + wr > prev:
                traffic[key] = rd + wr
        lines.append("")
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_ncu.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    out = [f"# launch lists ({args.tag})", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over one call inside a",
           "cudaProfilerStart/Stop window (tools/prof_bfs.py); shares of summed kernel time.", ""]
    for path in args.launches:
        rows = list(csv.reader(open(path)))
        h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        hdr = rows[h]
        ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = OrderedDict()
        for r in rows[h + 1:]:
            k = r[ki].split("(")[0].replace("void ", "").replace("gb::", "")[:60]
            t = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1e-9)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += t
        tot = sum(v[1] for v in agg.values()) or 1.0
        out.append(f"## {os.path.basename(path)} -- {len(rows) - h - 1} launches, {tot * 1e6:.1f} us")
        out.append("")
        out.append("| kernel | launches | us | share |")
        out.append("|---|---|---|---|")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            out.append(f"| {k} | {c} | {t * 1e6:.1f} | {t / tot:.1%} |")
        out.append("")
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_launches.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    for k, v in old.items():
        traffic.setdefault(k, v)
    with open(traffic_path, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
