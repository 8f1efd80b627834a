#!/bin/bash
# dev helper: the worldgen-bound configurations with the speculative pass as its own root vs behind k_step
for cfg in "--obs none" "--tier classic --obs none" "--obs pixels --max-episode-length 16"; do for r in 1 2; do for p in 0 1; do
  GR_SPEC_PDL=$p timeout 300 python bench.py $cfg --steps 300 --warmup 30 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$cfg] pdl=$p: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done; done
