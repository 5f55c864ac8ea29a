# per-level kernels of the host-driven loop (level 1 expand, level 2 pull) under ncu
export GFX_BFS_LOOP=host
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_lb_expand|k_bfs_pull|k_degree_scan" -c 4 -o gpurun_out/host_lv python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --warmup 1 > gpurun_out/ncu_host.log 2>&1
python tools/ncu_summary.py gpurun_out/host_lv.ncu-rep > gpurun_out/ncu_host_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/host_lv.ncu-rep 40 > gpurun_out/ncu_host_lines.txt 2>&1
python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --timing 2>&1 | tail -8 > gpurun_out/host_timing.txt
