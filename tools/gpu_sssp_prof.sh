timeout 300 python tools/prof_run.py --prim sssp --delta 4 --scale 24 --runs 1 --timing > gpurun_out/sssp4_timing.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp_persistent -c 1 -o gpurun_out/sssp4_full python tools/prof_run.py --prim sssp --delta 4 --scale 24 --runs 1 > gpurun_out/ncu_sssp4.log 2>&1
python tools/ncu_summary.py gpurun_out/sssp4_full.ncu-rep > gpurun_out/ncu_sssp4_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/sssp4_full.ncu-rep 40 > gpurun_out/ncu_sssp4_lines.txt 2>&1
head -30 gpurun_out/sssp4_timing.txt; grep -E "Duration|DRAM Through|L2 Cache Through|L1/TEX Cache Through|Issued Warp|No Eligible|Registers|Achieved Occ|dram__bytes" gpurun_out/ncu_sssp4_summary.txt; head -25 gpurun_out/ncu_sssp4_lines.txt
