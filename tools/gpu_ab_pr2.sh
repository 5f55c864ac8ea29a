for i in 1 2; do
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  echo -n "$lib "; python tools/pr_prof.py 24 20
done; done
unset GFX_LIB_PATH
timeout 600 python -m pytest tests/test_analytics_gpu.py tests/test_sssp_gpu.py -x -q 2>&1 | tail -1; python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
