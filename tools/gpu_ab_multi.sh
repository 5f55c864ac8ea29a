# bench-mode A/B of variant builds with N alternations (default 4):
#   bash tools/gpu_ab_multi.sh 4 base v1 v2   (paper_1701_01170_b200/libgfx_<name>.so)
n=$1; shift
for round in $(seq $n); do
for v in "$@"; do
  GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_$v.so python bench.py --no-extras --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import sys,json; d=json.loads(open('gpurun_out/ab_$v.json').read()); print('$v', d['value'], d['ms_per_step'], [round(l['ms']*1000,1) for l in d['roofline']['levels']])" 2>/dev/null || tail -2 gpurun_out/ab_$v.err
done; done | tee gpurun_out/ab_multi.txt
python - <<'PY'
import collections
d = collections.defaultdict(list)
for l in open('gpurun_out/ab_multi.txt'):
    p = l.split()
    if len(p) > 2:
        try: d[p[0]].append(float(p[2]))
        except ValueError: pass
for k, v in d.items():
    v.sort()
    print(f"{k}: median {v[len(v)//2]:.4f} ms  min {v[0]:.4f}  n={len(v)}")
PY
