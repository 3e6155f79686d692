#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
for w in 1 2 j1 j15; do
  timeout 300 python tools/small_calls.py $w > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/small_${w}_$TAG.csv python tools/small_calls.py $w > /dev/null 2>&1
  echo "== $w rc=$?"
  python - << PY
import csv
rows=list(csv.reader(open("gpurun_out/small_${w}_$TAG.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r)
H=rows[h]; ki,mi,vi,ii=(H.index(x) for x in ("Kernel Name","Metric Name","Metric Value","ID"))
d={}
for r in rows[h+1:]:
    if len(r)<=vi: continue
    d.setdefault(int(r[ii]),{"k":r[ki][:60]})[r[mi]]=r[vi]
ids=sorted(d); n=len(ids)//3
tot=0
for i in ids[-n:]:
    t=float(d[i]["gpu__time_duration.sum"])/1e3; tot+=t
    print(f"  {t:9.1f} us  grid {d[i]['launch__grid_size']:>8} x {d[i]['launch__block_size']:>4}  {d[i]['k']}")
print(f"  total {tot:.1f} us over {n} kernels (last call)")
PY
done
