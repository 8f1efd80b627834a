#!/bin/bash
# dev helper: side-stream priority on the default workload
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 300 --warmup 300 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "65536 [$v] "; python tools/dev/kt.py gpurun_out/ab.json
done
