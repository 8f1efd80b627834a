#!/bin/bash
# dev helper: delta e2e A/B -- huge-page host buffers and scatter prefetch distance
cat /sys/kernel/mm/transparent_hugepage/enabled; nproc
for r in 1 2; do
  for k in "GR_HOST_HUGE=0 GR_SCATTER_PF=0" "GR_HOST_HUGE=1 GR_SCATTER_PF=0" "GR_HOST_HUGE=0 GR_SCATTER_PF=16" "GR_HOST_HUGE=1 GR_SCATTER_PF=16" "GR_HOST_HUGE=1 GR_SCATTER_PF=48"; do
    env $k timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 40 2>/dev/null | grep "^{" > gpurun_out/e2e.json
    echo -n "$k: "; python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); e=d['e2e']; x=e['delta']
print('dense %.2fM' % (e['value']/1e6), 'delta %.2fM' % (x['value']/1e6), x['phases'])"
  done
done
