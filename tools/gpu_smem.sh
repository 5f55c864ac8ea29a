for pad in 0 9216 0 9216; do
  echo -n "pad=$pad "; GFX_SMEM_PAD=$pad python bench.py --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], [round(l['ms']*1000,1) for l in d['roofline']['levels']])"
done
