# A/B: HEAD build (libgfx_head.so) vs working tree build, same box, alternating
for i in 1 2 3; do
  echo -n "head  "; GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 5 2>&1 | grep device_ms
  echo -n "new   "; python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 5 2>&1 | grep device_ms
done
echo -n "head push "; GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 3 2>&1 | grep device_ms
echo -n "new  push "; python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 3 2>&1 | grep device_ms
