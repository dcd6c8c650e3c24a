"""One fused PPO rollout (16 envs x 300 steps) for ncu: python scripts/probe_ppo_rollout_ncu.py [--envs 16]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=16)
args = ap.parse_args()
rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=args.envs, master_seed=1)
tr = PPOTrainer(env, PPOConfig(rollout_steps=300, use_graph=False))
tr.rollout()
torch.cuda.synchronize()
print("ok")
