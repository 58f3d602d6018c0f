# Same-box A/B of library builds on the one-rank partitioned loops: bash tools/ab_dist.sh base l512
cd "${GRAFT_REPO_ROOT:-.}"
for v in "$@"; do echo "== $v"; GB_LIB=ab_lib/$v.so python tools/dist_loop_probe.py 24 | grep -v fused; done
