set -x
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "manual_learner or bias_grad or clip_adam or ppo or rows_to_bf16" 2>&1 | tail -15
for mb in 1 0; do
timeout 600 python -m paper_2402_16801_b200.ppo --total-timesteps 6553600 --manual-backward $mb 2>gpurun_out/ppo_mb$mb.log | tail -1
tail -2 gpurun_out/ppo_mb$mb.log
done
