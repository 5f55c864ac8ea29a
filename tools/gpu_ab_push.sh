# A/B of push-expansion variants: push-only BFS ms and SSSP ms (delta 4 / 32 /
# default) at s24 per build (paper_1701_01170_b200/libgfx_<name>.so)
for round in 1 2; do
for v in "$@"; do
  export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_$v.so
  echo "$v push $(python tools/bfs_push_time.py 2>&1 | tail -1) sssp $(python tools/sssp_time.py 2>&1 | tail -1)"
done; done
unset GFX_LIB_PATH
