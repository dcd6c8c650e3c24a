"""Time the fused rollout kernel from a mid-day state: ms per step of 2^20 envs."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup()
B, T, at = 1 << 20, 32, 128
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
pol = DeviceRandomPolicy(0, 16, 10)
pol.bind(range(B))
env.reset(as_numpy=False)
for _ in range(at):
    env.step(pol.actions(env), collect_infos=False)
obs = torch.empty(1, B, env.obs_length, device="cuda")
rew = torch.empty(1, B, device="cuda")
done = torch.empty(1, B, dtype=torch.uint8, device="cuda")
snap = {k: v.clone() for k, v in vars(env.states).items() if isinstance(v, torch.Tensor)}
ts = []
for rep in range(4):
    for k, v in snap.items():
        getattr(env.states, k).copy_(v)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    env.rollout(T, 0, pol.calls, obs, rew, done)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) / T)
print(f"rollout steps {at}..{at + T}: {min(ts[1:]):.4f} ms/step  ({B / min(ts[1:]) * 1e3:.3e} env-steps/s)")
