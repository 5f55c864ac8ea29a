GFX_BFS_WARPTIME=1 python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 2 2>&1 | grep -v "^ " | tail -20
