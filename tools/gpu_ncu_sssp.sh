# ncu --set full on the SSSP relax expansion (s24, delta 32): the heavy iterations
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lb_expand" --launch-skip 1 -c 3 -o gpurun_out/sssp_full python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 1 --warmup 0 > gpurun_out/ncu_sssp.log 2>&1
python tools/ncu_summary.py gpurun_out/sssp_full.ncu-rep > gpurun_out/ncu_sssp_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/sssp_full.ncu-rep 40 > gpurun_out/ncu_sssp_lines.txt 2>&1
python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 1 --timing 2>&1 | tail -20 > gpurun_out/sssp_timing.txt
