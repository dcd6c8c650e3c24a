"""Time the tcgen05 policy kernel alone at the C3 shape (4096 rows) and the
PPO rollout with / without it; --ncu runs a few launches for a profile."""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import ActorCritic, PPOConfig, PPOTrainer, pack_policy, policy_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--rows", type=int, default=4096)
args = ap.parse_args()
N = args.rows
net = ActorCritic(105, 17, 21, 64).cuda()
obs = torch.randn(N, 105, device="cuda")
ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
a = torch.zeros(N, 17, dtype=torch.uint8, device="cuda")
lp = torch.zeros(N, device="cuda")
v = torch.zeros(N, device="cuda")
with torch.no_grad():
    packed = pack_policy(net)
for _ in range(3):
    policy_step(obs, 105, 17, 21, packed, 1, ctr, a, lp, v)
torch.cuda.synchronize()
if args.ncu:
    sys.exit(0)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for s, e in ev:
    s.record()
    policy_step(obs, 105, 17, 21, packed, 1, ctr, a, lp, v)
    e.record()
torch.cuda.synchronize()
ts = sorted(s.elapsed_time(e) for s, e in ev)
flops = 2 * N * (128 * 112 + 2 * 64 * 64 + 416 * 64)
print(f"policy kernel {N} rows: median {1e3 * ts[len(ts) // 2]:.1f} us  ({flops / (ts[len(ts) // 2] / 1e3) / 1e12:.2f} TFLOP/s)")

rc = default_setup()
for fused in (True, False):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=4096, master_seed=1)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=300, fused_policy=fused))
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
    print(f"fused_policy={fused}: rollout {1e3 * (t1 - t0):.1f} ms  update {1e3 * (t2 - t1):.1f} ms")
    env.close()
