#!/bin/bash
# fused PPO rollout after the head / node-sum changes: parity (fused + wide), phases, timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ppo_rollout.py tests/test_gpu_wide.py tests/test_gpu_ppo.py -x -q -m gpu 2>&1 | tail -4
python scripts/probe_ppo_phases.py --envs 16 2>&1 | tail -12
for n in 16 512 2048; do timeout 300 python scripts/probe_ppo16.py --envs $n 2>&1 | tail -1; done
timeout 300 python scripts/probe_c1.py 2>&1 | tail -4
