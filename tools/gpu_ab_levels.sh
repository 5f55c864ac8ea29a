for d in auto push; do
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  echo "== $lib $d"; python tools/prof_run.py --prim bfs --direction $d --scale 24 --runs 1 --timing 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=ast.literal_eval(l); print(d['iteration'], d['mode'], round(d['ms']*1000,1), 'us')
    elif l.startswith('device_ms'): print(l[:60])
"
done; done
