"""Kernel-time breakdown of the PPO rollout's policy step (eager, 50 steps)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=4096, master_seed=1)
tr = PPOTrainer(env, PPOConfig(rollout_steps=50, use_graph=False))
tr.rollout()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.rollout()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
