# Round-2 evidence on one box: launch list of the bench command, one full ncu
# capture of k_bfs_persistent (s24 DO-BFS) and of the SSSP persistent loop.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-extras \
  --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "launch list rc $?"
bash tools/gpu_ncu_bfs.sh
echo "bfs ncu rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp_persistent -c 1 \
  -o gpurun_out/sssp_full python tools/prof_run.py --prim sssp --scale 24 --runs 1 --delta 4 \
  > gpurun_out/ncu_sssp.log 2>&1
python tools/ncu_summary.py gpurun_out/sssp_full.ncu-rep > gpurun_out/ncu_sssp_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/sssp_full.ncu-rep 40 > gpurun_out/ncu_sssp_lines.txt 2>&1
echo "sssp ncu rc $?"
