timeout 900 python -m pytest -q -x tests/test_parity_full_gpu.py::test_pagerank_full_vector tests/test_analytics_gpu.py tests/test_suite_gpu.py 2>&1 | tail -2
for r in 1 2 3; do
  echo "base $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/prof_run.py --prim pagerank --scale 24 --runs 3 --warmup 1 2>&1 | tail -1)"
  echo "prl1 $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_prl1.so python tools/prof_run.py --prim pagerank --scale 24 --runs 3 --warmup 1 2>&1 | tail -1)"
  echo "prh  $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_prh.so python tools/prof_run.py --prim pagerank --scale 24 --runs 3 --warmup 1 2>&1 | tail -1)"
done
