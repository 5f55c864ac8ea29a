for i in 1 2; do
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  for d in 32 1040; do
    echo -n "$lib delta=$d "; python tools/prof_run.py --prim sssp --delta $d --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
  done
done; done
unset GFX_LIB_PATH
timeout 900 python -m pytest tests/test_sssp_gpu.py tests/test_suite_gpu.py -x -q 2>&1 | tail -2
