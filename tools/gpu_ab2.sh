#!/bin/bash
# usage: bash tools/gpu_ab2.sh TAG "ENV=.. ENV=.." ... -- bench GEMM time + ncu DRAM bytes of the slice GEMM per env setting
TAG=$1; shift
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/ab_${TAG}_$i.json 2>/dev/null
  R=$(python -c "
import json; d=json.loads(open('gpurun_out/ab_${TAG}_$i.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), d['stages_ms']['ms_gemm'], d['clocks']['sm_mhz'])" 2>&1)
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"slicegemm_tc2" -s 1 -c 1 --csv --log-file gpurun_out/ab_${TAG}_$i.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
  N=$(python -c "
import csv
rows=list(csv.reader(open('gpurun_out/ab_${TAG}_$i.csv')))
h=next(i for i,r in enumerate(rows) if 'Metric Name' in r); H=rows[h]
mi,vi=H.index('Metric Name'),H.index('Metric Value')
d={r[mi]:r[vi] for r in rows[h+1:] if len(r)>vi}
print('ncu ms', round(float(d['gpu__time_duration.sum'])/1e6,2), 'DRAM rd GB', round(float(d['dram__bytes_read.sum'])/1e9,1), 'wr GB', round(float(d['dram__bytes_write.sum'])/1e9,1), 'hit', d['lts__t_sector_hit_rate.pct'], 'GHz', round(float(d['sm__cycles_elapsed.avg.per_second'])/1e9,3))" 2>&1)
  echo "[$cfg] step/gemm/MHz: $R | $N"
done
