#!/bin/bash
# dev helper: speculative pool knobs at a batch size (extended symbolic), 3 processes each
#   tools/dev/spec_sizes.sh <n_envs> "GR_SPEC=1 GR_WG_CTAS=1" ...
n=$1; shift
for v in "$@"; do for r in 1 2 3; do
  env $v timeout 300 python bench.py --envs $n --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'));print('n=$n [$v]', round(d['value']/1e6,2), d['ms_per_step'], {k: round(v/d['steps'],4) for k,v in d['kernel_ms'].items() if v})"
done; done
