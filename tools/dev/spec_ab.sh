B="python bench.py --e2e-steps 0 --no-cpu-baseline"
for cfg in "--tier classic --envs 1024" "--tier extended --envs 1024" "--tier extended --envs 4096" "--tier extended --envs 16384" "--tier extended --envs 65536" "--tier classic --obs pixels --envs 4096"; do
 for sp in 0 1; do
  echo -n "$cfg GR_SPEC=$sp: "; GR_SPEC=$sp timeout 600 $B $cfg --steps 300 --warmup 100 > gpurun_out/sp.json 2>gpurun_out/sp.err && python tools/dev/kt.py gpurun_out/sp.json | sed 's/gpurun_out.sp.json //' || tail -2 gpurun_out/sp.err
 done
done
