cat > /tmp/pr_time.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_1701_01170_b200.generators import rmat_device_graph
from paper_1701_01170_b200.primitives.pagerank import pagerank_device
from paper_1701_01170_b200.primitives.cc import cc_device
dg = rmat_device_graph(24, 16, 0)
for _ in range(2):
    r, st = pagerank_device(dg, 0.85, 0.0, 20)
print("pagerank s24 20it ms", round(st.device_ms, 3), "sum", float(r.sum()))
for _ in range(2):
    _, k, st = cc_device(dg)
print("cc s24 ms", round(st.device_ms, 3), "comps", k)
PY
for lib in head new; do
  if [ $lib = head ]; then export GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_head.so; else unset GFX_LIB_PATH; fi
  echo "== $lib"; python /tmp/pr_time.py
done
unset GFX_LIB_PATH
timeout 900 python -m pytest tests/test_analytics_gpu.py -x -q 2>&1 | tail -2
