# round evidence: GPU tests, default bench, reference arm, launch list, ncu of the persistent BFS
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --partitioned --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_part.json 2> gpurun_out/bench_part.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_ncu_bfs.sh
bash tools/gpu_ncu_sssp.sh
cat gpurun_out/pytest_gpu.txt
