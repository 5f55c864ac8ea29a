for i in 1 2; do
 echo -n "persist    "; python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
 echo -n "no persist "; GFX_NO_L2_PERSIST=1 python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
done
