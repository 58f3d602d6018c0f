cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2
NCU="ncu --clock-control none"
$NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2/launches_tc.csv python tools/prof_bfs.py --algo tc --scale 20 > /dev/null 2>&1
$NCU --profile-from-start off --set full --import-source on -k regex:tc_count -c 1 -o /tmp/r2_tc python tools/prof_bfs.py --algo tc --scale 20 > /dev/null 2>&1
ncu -i /tmp/r2_tc.ncu-rep --page raw --csv > gpurun_out/r2/full_tc.csv 2>/dev/null
ncu -i /tmp/r2_tc.ncu-rep --page source --csv > gpurun_out/r2/src_tc.csv 2>/dev/null
