#!/bin/bash
# dev helper: A/B classic-tier variants in lib/ab/ (symbolic at 1,024 and 65,536 envs)
for v in "$@"; do for a in "--envs 1024 --steps 300" "--steps 300"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py --tier classic --obs symbolic $a --warmup 50 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "$v $a: "; python tools/dev/kt.py gpurun_out/ab.json
done; done
