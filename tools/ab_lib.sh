# Same-box A/B of two library builds: ab_lib/base.so vs the in-tree build,
# alternating bench runs (device time per BFS), ROUNDS each.
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq ${ROUNDS:-3}); do
  for v in base cur; do
    if [ $v = base ]; then lib="GB_LIB=ab_lib/base.so"; else lib="GB_AB=cur"; fi
    env $lib $EXTRA timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-spmv --no-configs \
      > gpurun_out/abl_${v}_$r.json 2> gpurun_out/abl_${v}_$r.err
  done
done
python - <<'PY'
import glob, json
for v in ("base", "cur"):
    ms = []
    for f in sorted(glob.glob(f"gpurun_out/abl_{v}_*.json")):
        try:
            ms.append(json.loads(open(f).read().strip().splitlines()[-1])["ms_per_step"])
        except Exception as e:
            ms.append(None)
    print(v, ms)
PY
