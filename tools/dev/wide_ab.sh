#!/bin/bash
# dev helper: A/B the 256-thread extended worldgen (GR_WG_WIDE) at small batches
B="python bench.py --e2e-steps 0 --no-cpu-baseline"
for cfg in "--tier extended --envs 1024" "--tier extended --envs 4096" "--tier extended --obs pixels --envs 4096"; do
 for w in 0 1; do
  echo -n "$cfg GR_WG_WIDE=$w: "; GR_WG_WIDE=$w timeout 600 $B $cfg --steps 300 --warmup 100 > gpurun_out/ww.json 2>gpurun_out/ww.err && python tools/dev/kt.py gpurun_out/ww.json | sed 's/gpurun_out.ww.json //' || tail -2 gpurun_out/ww.err
 done
done
