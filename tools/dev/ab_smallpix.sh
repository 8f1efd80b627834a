#!/bin/bash
# dev helper: A/B lib/ab/ variants on the small-frame pixel configs (classic 7 / 10 px, extended 7 px), interleaved
for cfg in "--tier classic --tile-px 7" "--tier classic --tile-px 10" "--tier extended --tile-px 7"; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py $cfg --obs pixels --steps 300 --warmup 30 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$cfg] $v: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
