#!/bin/bash
# dev helper: A/B the library variants in lib/ab/ (interleaved, 2 rounds)
for r in 1 2; do
  for v in "$@"; do
    GR_LIB_VARIANT=$v timeout 300 python bench.py --steps 300 --warmup 300 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    echo -n "$v: "; python tools/dev/kt.py gpurun_out/ab.json
  done
done
