# Launch list (ncu, serialised) of one call of an algorithm on the host-driven
# engine:  bash tools/algo_launches.sh cc 24
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2
GB_BFS_GRAPH=0 GB_LOOP_GRAPH=0 ncu --clock-control none --profile-from-start off \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/r2/launches_$1.csv python tools/prof_bfs.py --algo $1 --scale $2 > /dev/null 2>&1
