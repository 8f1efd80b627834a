#!/bin/bash
# dev helper: GR_SPEC_REM_CTAS at the speculative-pool sizes, interleaved
for cfg in "--envs 1024" "--envs 4096" "--tier classic --envs 1024" "--tier classic"; do for r in 1 2; do for c in 0 148 32; do
  GR_SPEC_REM_CTAS=$c timeout 300 python bench.py $cfg --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$cfg] rem_ctas=$c: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done; done
