# ncu --set full of one PageRank round's kernels at s24
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_(gather|chunks|contrib|heavy)" -c 4 -o gpurun_out/pr_k python tools/pr_prof.py > gpurun_out/ncu_pr.log 2>&1
python tools/ncu_summary.py gpurun_out/pr_k.ncu-rep > gpurun_out/ncu_pr_summary.txt 2>&1
