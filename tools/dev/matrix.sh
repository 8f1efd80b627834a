#!/bin/bash
# dev helper: the SURVEY.md 8(d) configurations, one bench JSON each, into gpurun_out/matrix/
mkdir -p gpurun_out/matrix
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err; echo "$name rc=$?"; }
run ext_sym_65536 --steps 1000 --warmup 100
run reference_ext_sym_65536 --impl reference --steps 20 --warmup 5
run cls_sym_1024 --tier classic --envs 1024 --steps 1000 --warmup 100 --no-cpu-baseline
run cls_sym_65536 --tier classic --steps 1000 --warmup 100 --no-cpu-baseline
run cls_pix_4096 --tier classic --obs pixels --envs 4096 --steps 1000 --warmup 100 --no-cpu-baseline --e2e-steps 10
run cls_pix_65536 --tier classic --obs pixels --steps 500 --warmup 50 --no-cpu-baseline --e2e-steps 10
run ext_pix_65536 --obs pixels --steps 500 --warmup 50 --no-cpu-baseline --e2e-steps 10
run ext_pix_65536_L16 --obs pixels --max-episode-length 16 --steps 500 --warmup 50 --no-cpu-baseline --e2e-steps 10
for n in 1024 4096 16384 262144; do run ext_sym_$n --envs $n --steps 500 --warmup 50 --no-cpu-baseline --e2e-steps 10; done
run ext_sym_1048576 --envs 1048576 --steps 100 --warmup 10 --preroll 300 --no-cpu-baseline --e2e-steps 0
run ext_none_65536 --obs none --steps 1000 --warmup 100 --no-cpu-baseline --e2e-steps 10
run cls_none_65536 --tier classic --obs none --steps 1000 --warmup 100 --no-cpu-baseline --e2e-steps 10
GR_BENCH_BACKEND=gloo run gloo2_ext_sym_8192 --gpus 2 --envs 8192 --steps 50 --warmup 5 --preroll 50 --e2e-steps 3 --no-cpu-baseline
