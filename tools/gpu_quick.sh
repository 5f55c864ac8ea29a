# quick GPU iteration: BFS parity tests + a short bench (no extras)
timeout 600 python -m pytest tests/test_bfs_gpu.py tests/test_suite_gpu.py tests/test_analytics_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_quick.txt
timeout 600 python bench.py --no-extras --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
cat gpurun_out/pytest_quick.txt; tail -3 gpurun_out/bench_quick.err
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'init', d['roofline']['init_ms'])
for l in d['roofline']['levels']: print(l)
"
GFX_BFS_WARPTIME=1 python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 2>&1 | grep -v "^ " | tail -12
