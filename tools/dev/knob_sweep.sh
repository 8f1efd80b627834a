#!/bin/bash
# dev helper: env-knob A/B on the default workload, interleaved
#   tools/dev/knob_sweep.sh "" "GR_SPEC=1" "GR_WG_CTAS=3" ...
for r in 1 2; do
  for v in "$@"; do
    env $v timeout 300 python bench.py --steps 300 --warmup 300 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    echo -n "[$v]: "; python tools/dev/kt.py gpurun_out/ab.json
  done
done
