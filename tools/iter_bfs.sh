# quick BFS A/B on the GPU box: parity suite, then bench variants (env-selected)
timeout 600 python -m pytest tests/test_gpu_bfs.py -x -q > gpurun_out/t_bfs.log 2>&1
i=0
for v in ${VARIANTS:-"GB_BFS_ORDER=1" "GB_BFS_ORDER=1 GB_PUSH_MINB=1" "GB_BFS_ORDER=1 GB_PUSH_MINB=4" "GB_BFS_ORDER=0"}; do
  env $v timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-spmv > gpurun_out/b_v$i.json 2> gpurun_out/b_v$i.err
  echo "$v" > gpurun_out/b_v$i.name; i=$((i+1))
done
tail -3 gpurun_out/t_bfs.log
