#!/bin/bash
# dev helper: A/B lib/ab/ variants at several extended / classic symbolic sizes, interleaved
for n in 1024 4096 65536; do for r in 1 2; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py --envs $n --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "n=$n $v: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done; done
for r in 1 2; do for v in "$@"; do
  GR_LIB_VARIANT=$v timeout 300 python bench.py --tier classic --envs 1024 --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "classic n=1024 $v: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
