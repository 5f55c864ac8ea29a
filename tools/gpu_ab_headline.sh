# A/B of the headline DO-BFS: libgfx_head.so (HEAD build) vs the working tree,
# alternating runs on one box; then the BFS parity tests on the new build.
for i in 1 2 3; do
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  echo -n "$lib "; python bench.py --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['run']['per_call_ms'], d['roofline'].get('init_ms'), [round(l['ms']*1000,1) for l in d['roofline']['levels']])"
done; done
unset GFX_LIB_PATH
