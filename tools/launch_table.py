"""Print the per-launch durations of an ncu --metrics gpu__time_duration.sum
--csv log in launch order (one row per kernel launch).

    python tools/launch_table.py gpurun_out/warm_bfs.csv
"""
import csv
import sys

for path in sys.argv[1:]:
    hdr = None
    total = 0.0
    print(f"# {path}")
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) / 1e3
        total += us
        print(f"{d['Kernel Name'][:44]:44s} {d['Grid Size']:>14s} {us:9.1f} us")
    print(f"total {total:.1f} us")
