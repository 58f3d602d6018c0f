"""Side-by-side summary of `ncu -i rep --page raw --csv` exports (one kernel
per file, or every kernel row): duration, DRAM bytes, L2 sectors, hit
rates, sectors per request, occupancy and the top stall reasons."""
import csv
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("L2_rd_Msect", "lts__t_sectors_srcunit_tex_op_read.sum", 1e-6),
    ("L2_red_Msect", "lts__t_sectors_srcunit_tex_op_red.sum", 1e-6),
    ("L2_hit_pct", "lts__t_sector_hit_rate.pct", 1),
    ("L1_hit_pct", "l1tex__t_sector_hit_rate.pct", 1),
    ("ld_sect_per_req", "l1tex__average_t_sectors_per_request_pipe_lsu_mem_global_op_ld.ratio", 1),
    ("red_sect_per_req", "l1tex__average_t_sectors_per_request_pipe_lsu_mem_global_op_red.ratio", 1),
    ("shared_wavefronts_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
    ("occ_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
]
STALL = "smsp__average_warp_latency_issue_stalled_"


def load(path):
    with open(path) as f:
        r = list(csv.reader(f))
    hdr, units, data = r[0], r[1], r[2:]
    return hdr, data


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def summarize(path):
    hdr, data = load(path)
    out = []
    for row in data:
        d = {"kernel": row[hdr.index("Kernel Name")][:60]}
        for name, key, sc in KEYS:
            if key in hdr:
                v = num(row[hdr.index(key)])
                d[name] = None if v is None else round(v * sc, 2)
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = num(row[i])
                if v:
                    stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1
        d["stalls"] = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in stalls[:4])
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarize(p):
            print("##", p)
            for k, v in d.items():
                print(f"   {k:22s} {v}")
