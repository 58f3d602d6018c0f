# Same-box A/B of library builds in ab_lib/<name>.so (bench device time):
#   bash tools/ab_libs.sh base p4 p5
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq ${ROUNDS:-2}); do for v in "$@"; do
  GB_LIB=ab_lib/$v.so timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-spmv --no-configs \
    > gpurun_out/abx_${v}_$r.json 2> gpurun_out/abx_${v}_$r.err
done; done
for v in "$@"; do echo $v $(for r in $(seq ${ROUNDS:-2}); do python -c "import json; d=json.loads(open('gpurun_out/abx_${v}_$r.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], [x[2] for x in d['roofline']['level_ms'] if x[0]==2])" 2>/dev/null; done); done
