# grid-barrier cost and the DO-BFS barrier timeline (libgfx_timeline.so,
# built by: python tools/build_variant.py timeline -DGFX_BFS_TIMELINE)
python tools/gridsync_bench.py
GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_timeline.so python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 2 --warmup 2 2>&1 | tail -40
