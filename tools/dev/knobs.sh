#!/bin/bash
# dev helper: A/B the scheduling knobs (GR_WG_CTAS, GR_OBS_CTAS) on the default workload, interleaved
for r in 1 2; do
  for k in "GR_WG_CTAS=3" "GR_WG_CTAS=2" "GR_WG_CTAS=4" "GR_WG_CTAS=2 GR_OBS_CTAS=3" "GR_WG_CTAS=1"; do
    env $k timeout 300 python bench.py --steps 1000 --warmup 100 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/knob.json
    echo -n "$k: "; python tools/dev/kt.py gpurun_out/knob.json
  done
done
