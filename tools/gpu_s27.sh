# DO-BFS at scale 27 on one B200 (BASELINE config C5 input size, single GPU)
timeout 900 python tools/prof_run.py --prim bfs --direction auto --scale 27 --runs 3 --timing 2>&1 | tail -12
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
