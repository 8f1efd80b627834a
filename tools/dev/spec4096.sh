#!/bin/bash
# dev helper: repeated runs at 4,096 extended envs (bimodality of the speculative pool) per env setting
for v in "$@"; do for r in 1 2 3 4 5 6; do
  env $v timeout 300 python bench.py --envs 4096 --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['value']/1e6,2), d['ms_per_step'])"
done; done
