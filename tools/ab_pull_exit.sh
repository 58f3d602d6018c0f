#!/bin/bash
# Bounded row-bin pulls (cc_pull_exit / sssp_pull_exit, GB_PULL_EXIT=1) vs
# the edge-balanced tiles (GB_PULL_EXIT=0), same box, alternating:
# tools/time_algos.py device times.
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for e in 1 0; do
  echo "== GB_PULL_EXIT=$e r$r"
  GB_PULL_EXIT=$e timeout 600 python tools/time_algos.py --only ${ONLY:-cc,ccu,sssp} --reps 10
done; done
