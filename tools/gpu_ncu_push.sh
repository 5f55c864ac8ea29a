# ncu --set full of the host-loop push expansion kernels (push-only s24 BFS)
export GFX_BFS_LOOP=host
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lb_expand" -c 5 -o gpurun_out/push_lv python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 1 --warmup 1 > gpurun_out/ncu_push.log 2>&1
python tools/ncu_summary.py gpurun_out/push_lv.ncu-rep > gpurun_out/ncu_push_summary.txt 2>&1
python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 1 --timing 2>&1 | tail -10 > gpurun_out/push_host_timing.txt
unset GFX_BFS_LOOP
python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 2 --timing 2>&1 | tail -10 > gpurun_out/push_dev_timing.txt
