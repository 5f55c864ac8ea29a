# TC s22 per build (paper_1701_01170_b200/libgfx_<name>.so), two rounds
for round in 1 2; do
for v in "$@"; do
  echo "$v $(GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_$v.so python tools/tc_prof.py 22 2>&1 | tail -1)"
done; done
