"""Small lean + generic + rollout run for compute-sanitizer (memcheck / racecheck)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import EnvConfig, default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup(EnvConfig(episode_steps=24), days=30)
for B, dt in ((256, torch.float32), (100, torch.float64)):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=3, obs_dtype=dt)
    pol = DeviceRandomPolicy(seed=1, n_ports=env.n_ports, k=rc.env.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    for _ in range(30):
        env.step(pol.actions(env), collect_infos=False)
    print("mode", env.last_step_mode())
    if dt == torch.float32:
        obs = torch.empty(8, B, env.obs_length, device="cuda")
        rew = torch.empty(8, B, device="cuda")
        done = torch.empty(8, B, dtype=torch.uint8, device="cuda")
        env.rollout(8, 1, pol.calls, obs, rew, done)
    torch.cuda.synchronize()
    env.check_errors()
    env.close()
print("ok")
