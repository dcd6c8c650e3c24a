"""PPO at the paper's workload (16 envs, rollout 300, 4 x 4 minibatches):
rollout vs update time per iteration.  python scripts/probe_ppo16.py [--envs 16]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=16)
ap.add_argument("--per-step", action="store_true", help="the per-step policy + env pair, not vy_ppo_rollout")
args = ap.parse_args()
rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=args.envs, master_seed=1)
tr = PPOTrainer(env, PPOConfig(rollout_steps=300, fused_rollout=not args.per_step))
for _ in range(2):
    tr.iterate()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ro, up = [], []
for _ in range(5):
    ev[0].record()
    tr.rollout()
    ev[1].record()
    tr.update()
    ev[2].record()
    torch.cuda.synchronize()
    ro.append(ev[0].elapsed_time(ev[1]))
    up.append(ev[1].elapsed_time(ev[2]))
print(f"{tr.describe_rollout()[:40]}... envs {args.envs}: rollout {min(ro):.2f} ms ({min(ro) / 300 * 1e3:.1f} us/step), update {min(up):.2f} ms; "
      f"{(min(ro) + min(up)) / (300 * args.envs) * 1e5 / 1e3:.3f} s per 100k")
