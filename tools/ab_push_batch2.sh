#!/bin/bash
# Alternating same-box A/B of library builds in ab_lib/<name>.so (bench device
# time, 400 steps each); an argument may carry env settings after a colon:
#   bash tools/ab_push_batch2.sh b4 base b4:GB_PUSH_MINB=6
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq ${ROUNDS:-4}); do for spec in "$@"; do
  v=${spec%%:*}; e=""; [ "$spec" != "$v" ] && e=${spec#*:}
  tag=$(echo "$spec" | tr ':=' '__')
  env $e GB_LIB=ab_lib/$v.so timeout 300 python bench.py --steps 400 --no-cpu-baseline --no-spmv --no-configs \
    > gpurun_out/abq_${tag}_$r.json 2> gpurun_out/abq_${tag}_$r.err
  python -c "import json; d=json.loads(open('gpurun_out/abq_${tag}_$r.json').read().strip().splitlines()[-1]); print('$spec', $r, d['ms_per_step'], [x[2] for x in d['roofline']['level_ms'] if x[0]==1 and x[2] > 0.1])"
done; done
