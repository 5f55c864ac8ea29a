for k in 0 1 3; do
  echo "knobs=$k"; GFX_BFS_KNOBS=$k GFX_BFS_WARPTIME=1 python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 2 2>&1 | grep "warptime.*level 2\|phases.*level 2\|device_ms" | tail -3
done
timeout 600 python -m pytest tests/test_bfs_gpu.py -x -q 2>&1 | tail -2
