# Run on the GPU box (gpurun): bench lines, launch lists and ncu --set full
# captures of the hot kernels, all into gpurun_out/ (summarised into profiles/
# by tools/summarize_profiles.py).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --clock-control none"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# launch list of the bench command itself.  ncu cannot time kernels inside the
# conditional graph nodes, so this pass pins the host-driven engine (same kernels).
GB_BFS_GRAPH=0 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# one call of each algorithm inside a profiler window
for spec in "bfs 24" "cc 24" "pr 22" "sssp 20" "tc 20" "mxvm 24"; do
  set -- $spec
  GB_BFS_GRAPH=0 $NCU $( [ $1 = bfs ] && echo --cache-control none ) --profile-from-start off --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/launches_$1.csv python tools/prof_bfs.py --algo $1 --scale $2 > /dev/null 2>&1
done
# full captures of each algorithm's dominant kernel
GB_BFS_GRAPH=0 $NCU --profile-from-start off --set full --import-source on -k regex:bfs_expand -s 1 -c 1 \
  -o gpurun_out/prof_bfs python tools/prof_bfs.py --algo bfs --scale 24 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:mv_pull_tiles -c 1 \
  -o gpurun_out/prof_mxvm python tools/prof_bfs.py --algo mxvm --scale 24 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:pr_ -c 2 \
  -o gpurun_out/prof_pr python tools/prof_bfs.py --algo pr --scale 22 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:cc_ -c 3 \
  -o gpurun_out/prof_cc python tools/prof_bfs.py --algo cc --scale 24 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:"sssp_pull_tiles|lbs_expand" -c 3 \
  -o gpurun_out/prof_sssp python tools/prof_bfs.py --algo sssp --scale 20 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:tc_count -c 1 \
  -o gpurun_out/prof_tc python tools/prof_bfs.py --algo tc --scale 20 > /dev/null 2>&1
ls -la gpurun_out
