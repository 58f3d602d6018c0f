"""Summarise gpurun_out/b_v*.json bench variants (tools/iter_bfs.sh)."""
import glob
import json
import os

for f in sorted(glob.glob("gpurun_out/b_v*.json")):
    name = open(f[:-5] + ".name").read().strip() if os.path.exists(f[:-5] + ".name") else f
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(name, "FAILED", e)
        continue
    r = d["roofline"]
    print(f"{name:40s} {d['value']:8.1f} GTEPS {d['ms_per_step']:.4f} ms  push {r['launch_ms']:.4f} ms "
          f"frac {r['frac']:.3f}  levels {[round(t, 4) for (_k, _a, t) in r['level_ms']]}")
