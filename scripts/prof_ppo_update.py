import sys
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_01522_b200 import default_setup
from paper_2507_01522_b200.batch import BatchEnv
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer
rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=4096, master_seed=1)
tr = PPOTrainer(env, PPOConfig(rollout_steps=300))
tr.iterate(); torch.cuda.synchronize()
tr.rollout(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    tr.update(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
