#!/bin/bash
# dev helper: GR_SPEC on/off at mid batch sizes (extended symbolic), interleaved
for r in 1 2; do for n in 4096 8192 16384 32768; do for s in 0 1; do
  GR_SPEC=$s timeout 300 python bench.py --envs $n --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "n=$n GR_SPEC=$s: "; python tools/dev/kt.py gpurun_out/ab.json
done; done; done
