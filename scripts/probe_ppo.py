"""Split one PPO iteration (config C3: 4096 envs, 300-step rollout, 4x4
minibatch update) into rollout / update wall time on the device."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=4096, master_seed=1)
tr = PPOTrainer(env, PPOConfig(rollout_steps=300))
tr.iterate()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    tr.rollout()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tr.update()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rollout {1e3 * (t1 - t0):.1f} ms  update {1e3 * (t2 - t1):.1f} ms")
