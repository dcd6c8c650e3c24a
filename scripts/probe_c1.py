"""Config C1 (16 envs x 288-step episodes of the default station, random
policy) on the GPU: the fused rollout with the small-batch kernel (one warp
per env) and with the tile kernel, and the per-step public call, in
env-steps/s.  python scripts/probe_c1.py [--B 16] [--T 288]"""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--T", type=int, default=288)
args = ap.parse_args()
rc = default_setup()
B, T = args.B, args.T
for wide in (1, 0):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
    env.set_wide(wide)
    env.reset(as_numpy=False)
    obs = torch.empty(T, B, env.obs_length, device="cuda")
    rew = torch.empty(T, B, device="cuda")
    done = torch.empty(T, B, dtype=torch.uint8, device="cuda")
    env.rollout(T, 0, 0, obs, rew, done)  # warm-up
    ts = []
    for rep in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        env.rollout(T, 0, (rep + 1) * T, obs, rew, done)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = min(ts)
    print(f"rollout B={B} T={T} {'wide' if wide else 'tile'}: {ms:.3f} ms  {B * T / ms * 1e3:.3e} env-steps/s "
          f"({ms / T * 1e3:.2f} us/step)", flush=True)
    env.close()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
pol = DeviceRandomPolicy(0, env.n_ports, rc.env.discretization_k)
pol.bind(range(B))
env.reset(as_numpy=False)
for _ in range(10):
    env.step_random(pol)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(T):
    env.step_random(pol)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"step_random per call B={B}: {dt / T * 1e6:.1f} us/step  {B * T / dt:.3e} env-steps/s", flush=True)
