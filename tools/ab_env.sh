# Same-box A/B of env variants, alternating bench runs ROUNDS times:
#   bash tools/ab_env.sh "GB_X=0" "GB_X=1" ...
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq ${ROUNDS:-3}); do
  i=0
  for v in "$@"; do
    env $v timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-spmv --no-configs \
      > gpurun_out/abe_${i}_$r.json 2> gpurun_out/abe_${i}_$r.err
    i=$((i+1))
  done
done
python - "$@" <<'PY'
import glob, json, sys
for i, v in enumerate(sys.argv[1:]):
    ms, push = [], []
    for f in sorted(glob.glob(f"gpurun_out/abe_{i}_*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            ms.append(d["ms_per_step"]); push.append(d["roofline"]["launch_ms"])
        except Exception:
            ms.append(None)
    print(f"{v:40s} ms {ms} push {push}")
PY
