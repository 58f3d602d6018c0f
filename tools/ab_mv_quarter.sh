#!/bin/bash
# Masked pull SpMV medium rows: a half-warp per row (two rows a round trip)
# vs a quarter-warp per row (four), same box, alternating (tools/time_mv.py).
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in half quarter; do for u in "" "--uniform"; do
  echo "== $v $u r$r"; GB_LIB=ab_lib/$v.so timeout 300 python tools/time_mv.py --scale 24 --reps 20 $u | tail -1
done; done; done
