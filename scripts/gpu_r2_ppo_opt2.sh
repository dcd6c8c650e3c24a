#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ppo_rollout.py tests/test_gpu_ppo.py tests/test_gpu_policy*.py -x -q -m gpu 2>&1 | tail -4
python scripts/probe_ppo_phases.py --envs 16 2>&1 | tail -12
for n in 16 512 2048; do timeout 300 python scripts/probe_ppo16.py --envs $n 2>&1 | tail -1; done
for n in 16 4096; do timeout 300 python scripts/probe_ppo16.py --envs $n --per-step 2>&1 | tail -1; done
