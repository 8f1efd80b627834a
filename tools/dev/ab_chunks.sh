#!/bin/bash
# dev helper: A/B lib/ab/ variants on the e2e host transfers (symbolic dense + delta, pixels), interleaved
for r in 1 2; do for cfg in "--obs symbolic" "--obs pixels"; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py $cfg --steps 20 --warmup 5 --preroll 100 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);e=d['e2e']
print('[$cfg] $v dense', round(e['value']/1e6,2), e['phases']['ms_per_step'], 'delta', round(e.get('delta',{}).get('value',0)/1e6,2))"
done; done; done
