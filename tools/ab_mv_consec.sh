cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do
for v in base consec; do for rc in 0 1; do
  echo "== $v replay_consec=$rc r$r"; GB_REPLAY_CONSEC=$rc GB_LIB=ab_lib/$v.so timeout 200 python tools/time_mv.py --scale 24 --reps 20 2>&1 | tail -1
done; done; done
for rc in 0 1; do echo "== base uniform replay_consec=$rc"; GB_REPLAY_CONSEC=$rc GB_LIB=ab_lib/base.so timeout 200 python tools/time_mv.py --scale 24 --reps 20 --uniform 2>&1 | tail -1; done
