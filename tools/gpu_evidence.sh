# Round evidence on one box: GPU tests, default bench (all extras), launch list of
# the bench command, one ncu --set full capture of k_bfs_persistent (s24 DO-BFS).
# usage: bash tools/gpu_evidence.sh <tag>
t=${1:-r02b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${t}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${t}_launches.csv python bench.py --steps 2 --warmup 1 --no-extras \
  --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${t}_launches.csv > gpurun_out/${t}_launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bfs_persistent -c 1 \
  -o gpurun_out/${t}_bfs_full python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 \
  > gpurun_out/${t}_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/${t}_bfs_full.ncu-rep > gpurun_out/${t}_ncu_bfs_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${t}_bfs_full.ncu-rep 60 > gpurun_out/${t}_ncu_bfs_lines.txt 2>&1
cat gpurun_out/${t}_pytest_gpu.txt | tail -3
python - <<PY
import json; d=json.load(open('gpurun_out/${t}_bench.json'))
r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'frac', r['frac'], 'achieved', r['achieved'])
print('e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'))
for k,v in d.get('extras',{}).items(): print(' ', k, {kk: v.get(kk) for kk in ('gteps','ms','frac') if kk in v})
PY
head -30 gpurun_out/${t}_ncu_bfs_summary.txt
