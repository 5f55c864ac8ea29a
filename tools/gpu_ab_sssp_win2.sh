for r in 1 2 3; do
  echo "base $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_base.so python tools/sssp_time.py)"
  for w in 1 2 3 4; do echo "win$w $(GFX_SSSP_WIN=$w GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_win.so python tools/sssp_time.py)"; done
done
