# BFS A/B of env variants: bench (graph engine, device time) + warm launch list per variant
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_gpu_bfs.py -x -q > gpurun_out/t_bfs.log 2>&1
i=0
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-spmv --no-configs > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  env $v GB_BFS_GRAPH=0 timeout 300 ncu --cache-control none --clock-control none --profile-from-start off \
    --metrics gpu__time_duration.sum --csv --log-file gpurun_out/ab_$i.csv \
    python tools/prof_bfs.py --algo bfs --scale 24 --reps 2 > /dev/null 2>&1
  echo "$v" > gpurun_out/ab_$i.name; i=$((i+1))
done
tail -3 gpurun_out/t_bfs.log
