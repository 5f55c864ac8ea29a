timeout 600 python -m pytest tests/test_bfs_gpu.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; tail -3 gpurun_out/bench_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['ms_per_step'], json.dumps(d['e2e']))"
