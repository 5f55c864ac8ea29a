# full GPU test suite + default bench + launch list
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'frac', r['frac'], 'achieved', r['achieved'], 'traffic', r['traffic'])
print('e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'), 'extras', {k: v.get('gteps') for k,v in d.get('extras',{}).items()})
PY
