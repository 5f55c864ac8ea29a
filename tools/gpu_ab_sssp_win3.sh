timeout 900 python -m pytest -q -x tests/test_sssp_gpu.py tests/test_analytics_gpu.py tests/test_parity_full_gpu.py tests/test_dist_gpu.py -k "sssp" 2>&1 | tail -2
for r in 1 2; do
  echo "base"; GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/sssp_trace.py
  for w in 2 4 8; do echo "win$w"; GFX_SSSP_WIN=$w GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_win.so python tools/sssp_trace.py; done
done
