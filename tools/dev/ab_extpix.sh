#!/bin/bash
# dev helper: A/B lib/ab/ variants on extended pixels 10 px, 65,536 envs, interleaved
for r in 1 2; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py --obs pixels --steps 300 --warmup 30 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "$v: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
