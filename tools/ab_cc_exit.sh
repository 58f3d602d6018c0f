#!/bin/bash
# CC with the bounded row-bin pull (cc_pull_exit) vs the edge-balanced tiles
# (GB_CC_EXIT=0), same box, alternating: tools/time_algos.py device times.
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for e in 1 0; do
  echo "== GB_CC_EXIT=$e r$r"
  GB_CC_EXIT=$e timeout 600 python tools/time_algos.py --only cc,ccu --reps 10
done; done
