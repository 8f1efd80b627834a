#!/bin/bash
# dev helper: bench sweep over env-var knobs; each arg is "NAME=VAL,NAME=VAL"
for cfg in "$@"; do
  envs=$(echo "$cfg" | tr ',' ' ')
  env $envs timeout 300 python bench.py --steps 300 --warmup 300 --e2e-steps 0 --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  echo -n "$cfg: "; python tools/dev/kt.py gpurun_out/sw.json
done
