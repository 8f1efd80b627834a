#!/bin/bash
mkdir -p gpurun_out/ncu2
B="python bench.py --steps 3 --warmup 3 --preroll 400 --e2e-steps 0 --no-cpu-baseline"
cap() { name=$1; kern=$2; skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k $kern -s $skip -c 2 \
    -o gpurun_out/ncu2/$name $B "$@" > gpurun_out/ncu2/$name.log 2>&1; echo "$name rc=$?"; }
cap step k_step 390
cap worldgen k_worldgen 390
