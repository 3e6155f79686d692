#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_check.sh r2j
for it in 1 2; do for tb in 1 0; do
  MPCGEMM_PLANES_TB=$tb timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/tb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tb.json'));print('tb=$tb', round(d['ms_per_step'],2), d['stages_ms'])"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"linemax2|planes2" -c 4 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-extra 2>/dev/null | grep duration | awk -F'"' '{print $(NF-1), substr($10,1,40)}'
