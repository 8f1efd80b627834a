#!/bin/bash
# dev helper: the end-of-round ncu evidence: one `--set full` capture per hot
# kernel at steady state (two consecutive launches after a 400-step pre-roll)
# and the launch list of a short bench command.  One GPU, never multi-rank.
mkdir -p gpurun_out/ncu4
B="python bench.py --steps 3 --warmup 3 --preroll 400 --e2e-steps 0 --no-cpu-baseline"
cap() { name=$1; kern=$2; skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kern" -s $skip -c 2 \
    -o gpurun_out/ncu4/$name $B "$@" > gpurun_out/ncu4/$name.log 2>&1; echo "$name rc=$?"; }
cap sym '^k_symbolic_stage$' 800
cap step '^k_step$' 400
cap worldgen '^k_worldgen$' 800
cap pixels '^k_pixels$' 800 --obs pixels
cap pixprep '^k_pixprep$' 800 --obs pixels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/ncu4/launches.csv python bench.py --steps 20 --warmup 5 --preroll 30 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/ncu4/launches.log 2>&1; echo "launches rc=$?"
