#!/bin/bash
# dev helper: classic-tier scheduling knobs at 65,536 and 16,384 envs
B="python bench.py --e2e-steps 0 --no-cpu-baseline --tier classic"
for n in 65536 16384; do for kv in "GR_SPEC=0" "GR_SPEC=1" "GR_SPEC=1 GR_WG_CTAS=2" "GR_SPEC=0 GR_OBS_CTAS=1"; do
  echo -n "classic $n $kv: "; env $kv timeout 300 $B --envs $n --steps 300 --warmup 100 > gpurun_out/ck.json 2>/dev/null && python tools/dev/kt.py gpurun_out/ck.json | sed 's/gpurun_out.ck.json //'
done; done
