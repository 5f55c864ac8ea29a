# PageRank s24 (20 iterations, eps 0) per build: bash tools/gpu_ab_pr3.sh base v1 ...
for round in 1 2; do
for v in "$@"; do
  echo "$v $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_$v.so python tools/pr_time.py 2>&1 | tail -1)"
done; done
