for lib in libgfx.so libgfx_sssp_8_2.so libgfx_sssp_8_3.so libgfx_sssp_16_2.so; do
  for d in 32 0; do
    echo -n "$lib delta=$d "; GFX_LIB_PATH=$PWD/paper_1701_01170_b200/$lib python tools/prof_run.py --prim sssp --delta $d --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-40
  done
done
