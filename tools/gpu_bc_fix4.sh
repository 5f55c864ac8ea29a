timeout 1500 python -m pytest -q -x tests/test_analytics_gpu.py tests/test_suite_gpu.py tests/test_parity_full_gpu.py::test_bc_full_vector_s22_and_reproducible 2>&1 | tail -2
for r in 1 2 3; do
  echo "base $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/bc_prof.py 22)"
  echo "fix4 $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_fix4.so python tools/bc_prof.py 22)"
done
