for lib in libgfx.so libgfx_mb4.so libgfx_mb5.so libgfx.so; do
  echo -n "$lib "; GFX_LIB_PATH=$PWD/paper_1701_01170_b200/$lib python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
done
