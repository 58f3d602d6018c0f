# Same-box A/B of TC library builds: bash tools/ab_tc.sh base d16 ...
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in "$@"; do
  echo "$v $(GB_LIB=ab_lib/$v.so timeout 300 python tools/time_algos.py --only ${ALGO:-tc} 2>&1 | grep algo | tr "\n" " ")"
done; done
