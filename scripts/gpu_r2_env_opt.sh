#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ppo_rollout.py tests/test_gpu_wide.py -x -q -m gpu 2>&1 | tail -3
python scripts/probe_ppo_phases.py --envs 16 2>&1 | tail -22
timeout 300 python scripts/probe_ppo16.py --envs 16 2>&1 | tail -1
timeout 300 python scripts/probe_c1.py 2>&1 | tail -3
