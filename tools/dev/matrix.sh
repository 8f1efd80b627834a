#!/bin/bash
# dev helper: bench the section-8(d) configurations (device value, graph path)
B="python bench.py --e2e-steps 0 --no-cpu-baseline"
run() { echo -n "$*: "; timeout 600 $B "$@" > gpurun_out/mx.json 2>gpurun_out/mx.err && python tools/dev/kt.py gpurun_out/mx.json || tail -3 gpurun_out/mx.err; }
run --tier classic --obs symbolic --steps 300 --warmup 50
run --tier classic --obs symbolic --envs 1024 --steps 300 --warmup 50
run --tier classic --obs pixels --steps 200 --warmup 50
run --tier classic --obs none --steps 300 --warmup 50
run --tier extended --obs pixels --steps 200 --warmup 50
run --tier extended --obs symbolic --steps 300 --warmup 100
