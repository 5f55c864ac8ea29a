# PageRank s24: timing with the hub set at several sizes + ncu of the gather
for k in 0 8192 28672; do echo "hot=$k"; GFX_PR_HOT=$k timeout 300 python tools/prof_run.py --prim pagerank --scale 24 --runs 3 --warmup 1 2>&1 | tail -1; done > gpurun_out/pr_time.txt
timeout 600 ncu --set full --clock-control none -k regex:"k_pr_gather_hot|k_pr_contrib|k_pr_heavy" -c 3 -o gpurun_out/pr_full python tools/prof_run.py --prim pagerank --scale 24 --runs 1 --warmup 1 > gpurun_out/pr_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/pr_full.ncu-rep > gpurun_out/pr_ncu_summary.txt 2>&1
cat gpurun_out/pr_time.txt
