"""profiles/round2_ncu.md from gpurun_out/r2 (tools/collect_round2.sh):
per captured kernel the duration, DRAM bytes and % of peak, L2 / L1
throughput and hit rates, sectors per request for global loads and
reductions, occupancy, registers and the top stall reasons; then the
launch lists (kernel share of each algorithm call)."""
import csv
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_csv import num  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R2 = os.path.join(HERE, "gpurun_out", "r2")

COLS = [
    ("time", "gpu__time_duration.sum", "us"),
    ("dram rd", "dram__bytes_read.sum", "MB"),
    ("dram wr", "dram__bytes_write.sum", "MB"),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_active", ""),
    ("L2 rd sect", "lts__t_sectors_srcunit_tex_op_read.sum", "M"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", ""),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct", ""),
    ("ld sect/req", "ratio:l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum/"
                    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", ""),
    ("red sect/req", "ratio:l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum/"
                     "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", ""),
    ("occ %", "sm__warps_active.avg.pct_of_peak_sustained_active", ""),
    ("regs", "launch__registers_per_thread", ""),
]
UNIT = {"us": {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6,
               "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6},
        "MB": {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3},
        "M": {"sector": 1e-6, "": 1e-6}}


def conv(v, unit, want):
    x = num(v)
    if x is None:
        return "n/a"
    if want in UNIT:
        x *= UNIT[want].get(unit, 1)
    return f"{x:.1f}" if abs(x) >= 10 or x == 0 else f"{x:.2f}"


def cell(hdr, units, row, key, u):
    if key.startswith("ratio:"):
        a, b = key[6:].split("/")
        if a in hdr and b in hdr:
            x, y = num(row[hdr.index(a)]), num(row[hdr.index(b)])
            return f"{x / y:.2f}" if x is not None and y else "0 req"
        return "n/a"
    return conv(row[hdr.index(key)], units[hdr.index(key)], u) if key in hdr else "n/a"


def stalls(hdr, row):
    out = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            x = num(row[i])
            if x:
                out.append((x, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    out.sort(reverse=True)
    tot = sum(x for x, _ in out if _ != "selected") or 1
    return ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in out if n != "selected")[:90]


def full_tables():
    lines = []
    for path in sorted(glob.glob(os.path.join(R2, "full_*.csv"))):
        with open(path) as fh:
            r = list(csv.reader(fh))
        if len(r) < 3:
            continue
        hdr, units, rows = r[0], r[1], r[2:]
        lines.append(f"### {os.path.basename(path)[5:-4]}\n")
        lines.append("| kernel | " + " | ".join(c for c, _k, _u in COLS) + " | top stalls (excl. selected) |")
        lines.append("|" + "---|" * (len(COLS) + 2))
        for row in rows:
            k = row[hdr.index("Kernel Name")].split("(")[0][:48]
            cells = [cell(hdr, units, row, key, u) for _c, key, u in COLS]
            lines.append(f"| {k} | " + " | ".join(cells) + f" | {stalls(hdr, row)} |")
        lines.append("")
    return lines


def launch_tables():
    lines = []
    for path in sorted(glob.glob(os.path.join(R2, "launches_*.csv"))):
        with open(path) as fh:
            text = [ln for ln in fh if ln.startswith('"')]
        r = list(csv.reader(text))
        if not r:
            continue
        hdr = r[0]
        try:
            ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                              hdr.index("Metric Value"), hdr.index("Metric Unit"))
        except ValueError:
            continue
        per = {}
        order = []
        for row in r[1:]:
            if row[mi] != "gpu__time_duration.sum":
                continue
            k = row[ki].split("(")[0].replace("void ", "")[:40]
            t = num(row[vi]) * UNIT["us"].get(row[ui], 1)
            if k not in per:
                per[k] = [0, 0.0]
                order.append(k)
            per[k][0] += 1
            per[k][1] += t
        total = sum(v[1] for v in per.values()) or 1
        lines.append(f"### {os.path.basename(path)[9:-4]}: {sum(v[0] for v in per.values())} "
                     f"launches, {total:.0f} us of kernel time\n")
        lines.append("| kernel | launches | us | share |")
        lines.append("|---|---|---|---|")
        for k in sorted(order, key=lambda k: -per[k][1])[:14]:
            lines.append(f"| {k} | {per[k][0]} | {per[k][1]:.1f} | {100 * per[k][1] / total:.1f}% |")
        lines.append("")
    return lines


def main():
    out = ["# ncu summaries, round 2",
           "",
           "`tools/collect_round2.sh` on one B200 (`ncu --clock-control none`, serialised, "
           "cold caches between kernel replays); host-driven engines so the kernels launch "
           "outside conditional graph nodes. Times here are per launch under the profiler, "
           "not bench values.",
           "", "## Full captures (`--set full`)", ""]
    out += full_tables()
    out += ["## Launch lists (one call of each algorithm)", ""]
    out += launch_tables()
    dst = os.path.join(HERE, "profiles", "round2_ncu.md")
    with open(dst, "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()
