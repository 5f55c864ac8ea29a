# DO-BFS with different L1/shared carveouts (percent shared) for k_bfs_persistent
for cv in none 50 60 75 100 50 none; do
  if [ $cv = none ]; then unset GFX_BFS_CARVEOUT; else export GFX_BFS_CARVEOUT=$cv; fi
  echo -n "carveout $cv "; python bench.py --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], [round(l['ms']*1000,1) for l in d['roofline']['levels']])"
done
unset GFX_BFS_CARVEOUT
