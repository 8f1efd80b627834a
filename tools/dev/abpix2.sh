#!/bin/bash
# dev helper: A/B pixel variants (ext px10 65,536 envs and classic px7 65,536 envs), interleaved
for r in 1 2; do for v in "$@"; do
  for cfg in "--tier extended" "--tier classic"; do
    GR_LIB_VARIANT=$v timeout 300 python bench.py $cfg --obs pixels --steps 200 --warmup 20 --preroll 200 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    echo -n "$v $cfg: "; python tools/dev/kt.py gpurun_out/ab.json
  done
done; done
