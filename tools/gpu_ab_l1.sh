timeout 900 python -m pytest -q -x tests/test_bfs_gpu.py tests/test_analytics_gpu.py 2>&1 | tail -2
bash tools/gpu_ab_multi.sh 5 base l1 2>&1 | tail -2
for r in 1 2 3; do
  echo "base $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/bc_prof.py 22)"
  echo "l1   $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_l1.so python tools/bc_prof.py 22)"
done
