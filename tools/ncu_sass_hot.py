"""Top SASS instructions of one kernel in an ncu report by warp-stall samples
and by executed instructions (ncu --page source --print-source sass).

    python tools/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:])))
        if (r.get("# Samples") or "").isdigit()]
tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
tot_i = sum(int(r["Instructions Executed"] or 0) for r in rows)
print(f"{len(rows)} SASS lines, {tot_s} stall samples, {tot_i} warp instructions")
for i, r in enumerate(rows):
    r["_pos"] = i
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
for r in sorted(hot, key=lambda r: r["_pos"]):
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{r['_pos']:5d} {100*s/max(tot_s,1):5.1f}%  ex={int(r['Instructions Executed'] or 0):>10d}  {r['Source'].strip()[:70]}")
