#!/bin/bash
# dev helper: speculative pool (now a programmatic dependent of k_step) on/off across configurations
for cfg in "--envs 16384" "--envs 32768" "--envs 65536" "--obs pixels --tier classic --envs 4096" "--obs pixels --tier classic" "--obs pixels --envs 16384"; do for s in 0 1; do
  GR_SPEC=$s timeout 300 python bench.py $cfg --steps 300 --warmup 30 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$cfg] spec=$s: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
