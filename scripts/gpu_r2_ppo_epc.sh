#!/bin/bash
# fused PPO rollout: parity, then rollout time vs envs per CTA (VY_PPO_EPC)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ppo_rollout.py -x -q -m gpu 2>&1 | tail -4
for n in 16 64 512 2048; do
  for e in 16 8 4 2 1; do
    echo "epc $e"; VY_PPO_EPC=$e timeout 300 python scripts/probe_ppo16.py --envs $n 2>&1 | tail -1
  done
done
