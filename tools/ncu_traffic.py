"""profiles/ncu_traffic.json from the ncu --set full captures of
tools/collect_round2.sh (gpurun_out/r2/full_*.csv): DRAM bytes read + written
per launch of each captured kernel (the largest launch of a kernel name; the
uniform masked SpMV sums its stripe launches into one call).  bench.py reads
it for the `traffic` field of its roofline objects."""
import csv
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_csv import num  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R2 = os.path.join(HERE, "gpurun_out", "r2")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    out = {"_source": "round 2: profiles/round2_ncu.md (tools/collect_round2.sh), "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch (tools/ncu_traffic.py)"}
    for path in sorted(glob.glob(os.path.join(R2, "full_*.csv"))):
        tag = os.path.basename(path)[5:-4]
        with open(path) as fh:
            r = list(csv.reader(fh))
        if len(r) < 3:
            continue
        hdr, units, rows = r[0], r[1], r[2:]
        rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        per = {}
        for row in rows:
            name = row[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "")
            name = name.replace("gb::", "").strip()
            b = num(row[rd]) * SCALE.get(units[rd], 1) + num(row[wr]) * SCALE.get(units[wr], 1)
            per.setdefault(name, []).append(b)
        for name, bs in per.items():
            if tag == "mxvm_u" and name == "mv_pull_binned":
                out["mv_pull_binned_uniform_striped"] = float(sum(bs))
            else:
                out[name] = max(float(max(bs)), out.get(name, 0.0))
    dst = os.path.join(HERE, "profiles", "ncu_traffic.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print("wrote", dst, len(out) - 1, "kernels")


if __name__ == "__main__":
    main()
