#!/bin/bash
# dev helper: A/B library variants in lib/ab/ at small and default batches
B="python bench.py --e2e-steps 0 --no-cpu-baseline"
for cfg in "--tier extended --envs 1024" "--tier classic --envs 1024" "--tier extended --envs 65536"; do
 for v in "$@"; do
  echo -n "$cfg $v: "; GR_LIB_VARIANT=$v timeout 600 $B $cfg --steps 300 --warmup 100 > gpurun_out/abs.json 2>gpurun_out/abs.err && python tools/dev/kt.py gpurun_out/abs.json | sed 's/gpurun_out.abs.json //' || tail -2 gpurun_out/abs.err
 done
done
