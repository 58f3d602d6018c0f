cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in base t8 t32; do
  GB_LIB=ab_lib/$v.so timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-spmv --no-configs > gpurun_out/ab3_${v}_$r.json 2>gpurun_out/ab3_${v}_$r.err
done; done
for v in base t8 t32; do echo $v $(for r in 1 2; do python -c "import json,sys; d=json.loads(open('gpurun_out/ab3_${v}_$r.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['launch_ms'])" 2>/dev/null; done); done
