#!/bin/bash
# dev helper: e2e through BatchEnv.step at several sizes, compact transfer on / off
for cfg in "--envs 65536" "--envs 16384" "--envs 4096" "--obs pixels --envs 65536" "--tier classic --envs 65536" "--tier classic --obs pixels --envs 65536"; do
  for c in 1 0; do
    GR_HOST_COMPACT=$c timeout 300 python bench.py $cfg --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 20 2>/dev/null | grep "^{" > gpurun_out/e2e.json
    echo -n "$cfg compact=$c: "; python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); e=d['e2e']; x=e.get('delta') or {}
print('dense %.2fM' % (e['value']/1e6), e['phases']['ms_per_step'], 'delta %.2fM' % (x.get('value', 0)/1e6))"
  done
done
