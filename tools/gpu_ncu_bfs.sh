# one ncu --set full capture of the persistent DO-BFS kernel at s24 + summaries
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bfs_persistent -c 1 -o gpurun_out/bfs_full python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/bfs_full.ncu-rep > gpurun_out/ncu_bfs_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/bfs_full.ncu-rep 60 > gpurun_out/ncu_bfs_lines.txt 2>&1
