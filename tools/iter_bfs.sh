timeout 600 python -m pytest tests/test_gpu_bfs.py -x -q > gpurun_out/t_bfs.log 2>&1
for o in 0 1; do GB_BFS_ORDER=$o timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-spmv > gpurun_out/b_order$o.json 2> gpurun_out/b_order$o.err; done
GB_BFS_GRAPH=0 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:bfs_expand -s 1 -c 1 -o gpurun_out/r2_push_smem3 python tools/prof_bfs.py --scale 24 > gpurun_out/ncu_push.log 2>&1
GB_BFS_ORDER=0 GB_BFS_GRAPH=0 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:bfs_expand -s 1 -c 1 -o gpurun_out/r2_push_warp3 python tools/prof_bfs.py --scale 24 > gpurun_out/ncu_push.log 2>&1
tail -3 gpurun_out/t_bfs.log
