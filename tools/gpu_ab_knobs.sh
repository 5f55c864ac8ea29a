# A/B of a knob in bench mode (same build)
for i in 1 2; do
for k in 0 1; do
  echo -n "knobs=$k "; GFX_BFS_KNOBS=$k python bench.py --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('init_ms'), [round(l['ms']*1000,1) for l in d['roofline']['levels']])"
done; done
timeout 600 python -m pytest tests/test_bfs_gpu.py -x -q 2>&1 | tail -2
