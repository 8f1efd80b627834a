B="python bench.py --e2e-steps 0 --no-cpu-baseline"
for cfg in "--obs pixels" "--obs none" "--tier classic"; do for w in 0 3 2; do
  echo -n "$cfg WG=$w: "; GR_WG_CTAS=$w timeout 600 $B $cfg --steps 300 --warmup 100 > gpurun_out/sw2.json 2>/dev/null && python tools/dev/kt.py gpurun_out/sw2.json | sed 's/gpurun_out.sw2.json //'
done; done
