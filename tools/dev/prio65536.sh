#!/bin/bash
# dev helper: env settings on the default workload (default steps / warm-up), interleaved
for r in 1 2 3 4; do for v in "$@"; do
  env $v timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "65536 [$v] "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
