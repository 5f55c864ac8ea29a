for mb in 1 4 6 8; do
  echo -n "minb=$mb "; GFX_BFS_LOOP=host GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_pull$mb.so python tools/prof_run.py --prim bfs --direction auto --scale 24 --runs 1 --timing 2>&1 | grep "'iteration': [23]" | python -c "
import sys,ast
print([round(ast.literal_eval(l.strip())['ms']*1000,1) for l in sys.stdin])"
done
