# Round-2 evidence, run on the GPU box (gpurun): launch lists and ncu --set
# full captures of every hot kernel, exported as raw CSV into gpurun_out/
# (summarised into profiles/round2_ncu.md by tools/summarize_round2.py).
# The device loops (BFS / SSSP / PR / CC) run inside conditional graph nodes,
# which ncu does not enumerate: these captures pin the host-driven engines
# (GB_BFS_GRAPH=0, GB_LOOP_GRAPH=0) -- the same kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r2
NCU="ncu --clock-control none"
export GB_BFS_GRAPH=0 GB_LOOP_GRAPH=0
# launch list of one BFS (bench workload) and of each algorithm
for spec in "bfs 24" "mxvm 24" "pr 22" "cc 24" "sssp 20" "tc 20" "push 24" "mxm 20"; do
  set -- $spec
  $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file gpurun_out/r2/launches_$1.csv python tools/prof_bfs.py --algo $1 --scale $2 > /dev/null 2>&1
done
cap() {  # name regex algo scale count
  $NCU --profile-from-start off --set full -k regex:"$2" -c $5 -o /tmp/r2_$1 \
    python tools/prof_bfs.py --algo $3 --scale $4 > /dev/null 2>&1
  ncu -i /tmp/r2_$1.ncu-rep --page raw --csv > gpurun_out/r2/full_$1.csv 2>/dev/null
}
cap bfs_push "bfs_expand_warp" bfs 24 2
cap bfs_pull "bfs_pull" bfs 24 1
cap mxvm "mv_pull_binned" mxvm 24 1
cap mxvm_u "mv_pull_binned" mxvm_u 24 3   # uniform: column stripes (3 launches)
cap pr "pr_spmv|pr_epilogue" pr 22 2
cap cc "cc_pull|cc_hook|cc_shortcut" cc 24 5   # cc_pull matches cc_pull_exit
cap sssp "sssp_pull|lbs_expand" sssp 20 5   # tiles, the bounded bins (sssp_pull_exit), push
cap tc "tc_count" tc 20 1
cap push "lbs_expand" push 24 1
cap mxm "mxm_masked_kernel" mxm 20 1
ls -la gpurun_out/r2
