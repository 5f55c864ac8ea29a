# A/B in bench mode: HEAD build (libgfx_head.so) vs working tree, alternating
for i in 1 2 3; do
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  echo -n "$lib "; python bench.py --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['per_call_ms'], d['roofline'].get('init_ms'), [round(l['ms']*1000,1) for l in d['roofline']['levels']])"
done; done
unset GFX_LIB_PATH
timeout 900 python -m pytest tests/test_bfs_gpu.py tests/test_dist_gpu.py tests/test_suite_gpu.py tests/test_operators_gpu.py -x -q 2>&1 | tail -2
