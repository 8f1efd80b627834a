#!/bin/bash
# dev helper: side-stream priority vs the classic 65,536-env schedule (repeated processes)
for r in 1 2 3 4; do for v in "GR_SIDE_PRIO=-1" "GR_SIDE_PRIO=1" "GR_SIDE_PRIO=0"; do
  env $v timeout 300 python bench.py --tier classic --steps 500 --warmup 50 --preroll 400 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  echo -n "[$v]: "; python tools/dev/kt.py gpurun_out/ab.json | sed "s/{.*}//"
done; done
