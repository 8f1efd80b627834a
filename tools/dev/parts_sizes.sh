#!/bin/bash
# dev helper: GR_INSTALL_PARTS at several extended sizes, interleaved
for n in 8192 16384 32768; do for r in 1 2; do for p in 1 4; do
  GR_INSTALL_PARTS=$p timeout 300 python bench.py --envs $n --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "n=$n parts=$p: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done; done
