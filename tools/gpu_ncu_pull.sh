# ncu --set full of the host-loop pull kernels (levels 2-4 of the s24 DO-BFS)
export GFX_BFS_LOOP=host
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_pull" -c 3 -o gpurun_out/pull_lv python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --warmup 1 > gpurun_out/ncu_pull.log 2>&1
python tools/ncu_summary.py gpurun_out/pull_lv.ncu-rep > gpurun_out/ncu_pull_summary.txt 2>&1
python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --timing 2>&1 | tail -8 > gpurun_out/pull_host_timing.txt
