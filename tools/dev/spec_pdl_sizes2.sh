#!/bin/bash
# dev helper: speculative pool on/off, extended pixels and symbolic mid sizes
for cfg in "--obs pixels --envs 65536" "--obs pixels --envs 4096" "--envs 8192" "--envs 24576"; do for s in 0 1; do
  GR_SPEC=$s timeout 300 python bench.py $cfg --steps 300 --warmup 30 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$cfg] spec=$s: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
