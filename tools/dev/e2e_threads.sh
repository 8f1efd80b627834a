#!/bin/bash
# dev helper: e2e (compact dense + delta) vs host thread count
for r in 1 2; do for t in 16 12 8 6; do
  GR_HOST_THREADS=$t timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 40 2>/dev/null | grep "^{" > gpurun_out/e2e.json
  echo -n "threads $t: "; python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); e=d['e2e']; x=e['delta']
print('dense %.2fM' % (e['value']/1e6), e['phases']['ms_per_step'], 'delta %.2fM' % (x['value']/1e6), x['phases']['ms_per_step'])"
done; done
