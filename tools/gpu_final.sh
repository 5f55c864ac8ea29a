# final evidence: GPU tests, smoke, default bench, partitioned bench, reference arm,
# launch list of the bench, ncu --set full of the persistent BFS and SSSP kernels
set -x
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --partitioned --no-cpu-baseline --no-e2e > gpurun_out/bench_part.json 2> gpurun_out/bench_part.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_ncu_bfs.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp_persistent -c 1 -o gpurun_out/sssp4_full python tools/prof_run.py --prim sssp --delta 4 --scale 24 --runs 1 > gpurun_out/ncu_sssp4.log 2>&1
python tools/ncu_summary.py gpurun_out/sssp4_full.ncu-rep > gpurun_out/ncu_sssp4_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/sssp4_full.ncu-rep 40 > gpurun_out/ncu_sssp4_lines.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt
