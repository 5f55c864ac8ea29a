python tools/bc_prof.py 22
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bc_launches.csv python tools/bc_prof.py 22 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/bc_launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[i]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
ks=[(r[ki][:50], float(r[vi].replace(',',''))*(1e-3 if r[ui]=='ns' else 1)) for r in rows[i+1:]]
# last BC call: find last occurrence of k_bc_seed
last=max(j for j,(k,_) in enumerate(ks) if 'k_bc_seed' in k)
start=max(j for j,(k,_) in enumerate(ks[:last]) if 'k_bc_accumulate' in k)+1
seg=ks[start:]
tot=collections.defaultdict(float); cnt=collections.Counter()
for k,t in seg: tot[k]+=t; cnt[k]+=1
print('launches', len(seg), 'sum us', round(sum(t for _,t in seg),1))
for k,t in sorted(tot.items(), key=lambda x:-x[1]): print(f'{t:9.1f} us  x{cnt[k]:3d}  {k}')
PY
