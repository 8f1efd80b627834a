#!/bin/bash
# dev helper: A/B pixel variants in lib/ab/
for r in 1 2; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py --tier extended --obs pixels --steps 200 --warmup 50 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "$v: "; python tools/dev/kt.py gpurun_out/ab.json
done; done
