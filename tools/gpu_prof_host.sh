# per-level kernels of one DO-BFS (host level loop) under ncu --set full
export GFX_BFS_LOOP=host
timeout 900 ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/bfs_host_full python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --warmup 1 > gpurun_out/ncu_host.log 2>&1
python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 3 --timing > gpurun_out/host_timing.log 2>&1
