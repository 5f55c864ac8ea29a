# SSSP two-level far pile: parity tests, then A/B of window widths against the one-pile build
timeout 900 python -m pytest -q -x tests/test_sssp_gpu.py tests/test_analytics_gpu.py -k "sssp" 2>&1 | tail -2
for r in 1 2 3; do
  echo "base $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/sssp_time.py)"
  for w in 4 8 16 32; do echo "win$w $(GFX_SSSP_WIN=$w GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_win.so python tools/sssp_time.py)"; done
done
