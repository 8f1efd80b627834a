#!/bin/bash
# dev helper: one `ncu --set full` capture of a kernel at steady state
#   tools/dev/ncu_one.sh <name> <kernel-regex> <launch-skip> [bench args...]
mkdir -p gpurun_out/ncu3
name=$1; kern=$2; skip=$3; shift 3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kern -s $skip -c 2 \
  -o gpurun_out/ncu3/$name python bench.py --steps 3 --warmup 3 --preroll 200 --e2e-steps 0 --no-cpu-baseline "$@" \
  > gpurun_out/ncu3/$name.log 2>&1
echo "$name rc=$?"
