#!/bin/bash
# Same-box A/B of the push batch per round trip (GB_WT_B) and its register
# budget (GB_PUSH_MINB): bench device time and the level-2 push launch.
cd "${GRAFT_REPO_ROOT:-.}"
run() {  # tag lib env...
  local tag=$1 lib=$2; shift 2
  env "$@" GB_LIB=ab_lib/$lib.so timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-spmv --no-configs \
    > gpurun_out/abp_$tag.json 2> gpurun_out/abp_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/abp_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['ms_per_step'], [x[2] for x in d['roofline']['level_ms'] if x[0]==1 and x[2] > 0.1])"
}
for r in $(seq ${ROUNDS:-2}); do
  run base_$r base GB_PUSH_MINB=5
  run b16_$r b16 GB_PUSH_MINB=5
  run b16m4_$r b16 GB_PUSH_MINB=4
  run b4_$r b4 GB_PUSH_MINB=5
done
