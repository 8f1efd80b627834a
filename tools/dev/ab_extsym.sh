#!/bin/bash
# dev helper: extended symbolic writer shapes on the default workload (lib variant + env knobs), interleaved
for r in 1 2; do for v in "w2 X=0" "w1 GR_OBS_CTAS=4 GR_OBS_CTAS0=6" "w1 GR_OBS_CTAS=5 GR_OBS_CTAS0=6" "w1 GR_OBS_CTAS=3 GR_OBS_CTAS0=6"; do
  set -- $v; lib=$1; shift
  env GR_LIB_VARIANT=$lib "$@" timeout 300 python bench.py --steps 300 --warmup 300 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$v]: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
