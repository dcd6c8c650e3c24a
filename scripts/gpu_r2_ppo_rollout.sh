#!/bin/bash
# fused PPO rollout: parity tests, the PPO/wide suites it touches, smoke, PPO(16) timing both ways
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ppo_rollout.py tests/test_gpu_ppo.py tests/test_gpu_wide.py -x -q -m gpu 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
for n in 16 64 512 2048; do
  timeout 300 python scripts/probe_ppo16.py --envs $n 2>&1 | tail -1
  timeout 300 python scripts/probe_ppo16.py --envs $n --per-step 2>&1 | tail -1
done
