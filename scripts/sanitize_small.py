"""Small runs of every step-kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): lean + generic steps, the fused policy
step, the rollout (ragged tile, episode boundary), the streamed C4 tile and
the one-launch heterogeneous kernel."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import EnvConfig, default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups  # noqa: E402
from paper_2507_01522_b200.workloads import c4_setup  # noqa: E402

rc = default_setup(EnvConfig(episode_steps=24), days=30)
for B, dt in ((256, torch.float32), (100, torch.float64)):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=3, obs_dtype=dt)
    pol = DeviceRandomPolicy(seed=1, n_ports=env.n_ports, k=rc.env.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    for _ in range(30):
        env.step(pol.actions(env), collect_infos=False)
    print("mode", env.last_step_mode())
    for _ in range(5):
        env.step_random(pol)
    if dt == torch.float32:
        obs = torch.empty(30, B, env.obs_length, device="cuda")
        rew = torch.empty(30, B, device="cuda")
        done = torch.empty(30, B, dtype=torch.uint8, device="cuda")
        env.rollout(30, 1, pol.calls, obs, rew, done)  # crosses the episode end
    torch.cuda.synchronize()
    env.check_errors()
    env.close()
# rollouts with a ragged last tile: the tile kernel and the one-warp-per-env kernel; wide single steps
for wide in (0, 1):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=77, master_seed=4)
    env.set_wide(wide)
    env.reset(as_numpy=False)
    obs = torch.empty(30, 77, env.obs_length, device="cuda")
    rew = torch.empty(30, 77, device="cuda")
    done = torch.empty(30, 77, dtype=torch.uint8, device="cuda")
    env.rollout(30, 2, 0, obs, rew, done)
    print("rollout mode", env.last_step_mode())
    torch.cuda.synchronize()
    env.close()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=64, master_seed=4)
env.set_wide(1)
pol = DeviceRandomPolicy(seed=1, n_ports=env.n_ports, k=rc.env.discretization_k)
pol.bind(range(64))
env.reset(as_numpy=False)
for _ in range(30):
    env.step(pol.actions(env), collect_infos=False)
print("step mode", env.last_step_mode())
torch.cuda.synchronize()
env.close()
# streamed C4 tile (ragged), episode boundary
c4 = c4_setup(days=20)
cfg = EnvConfig(battery_enabled=True, alpha=c4.env.alpha, beta=c4.env.beta, episode_steps=12)
env = BatchEnv(cfg, c4.station, c4.dataset, batch_size=70, master_seed=5)
pol = DeviceRandomPolicy(seed=2, n_ports=env.n_ports, k=cfg.discretization_k)
pol.bind(range(70))
env.reset(as_numpy=False)
for _ in range(15):
    env.step_random(pol)
print("mode", env.last_step_mode())
torch.cuda.synchronize()
env.close()
# streamed C4 tile with its L2 prefetch of later tiles active (40 tiles; run with VY_PF=10 so the
# prefetch distance is a few tiles at this size)
env = BatchEnv(cfg, c4.station, c4.dataset, batch_size=1280, master_seed=6)
pol = DeviceRandomPolicy(seed=3, n_ports=env.n_ports, k=cfg.discretization_k)
pol.bind(range(1280))
env.reset(as_numpy=False)
for _ in range(6):
    env.step_random(pol)
print("mode", env.last_step_mode())
torch.cuda.synchronize()
env.close()
# one-launch heterogeneous batch (ragged last group)
groups = sweep_groups(36 * 32 + 7, days=20)[:6]
for g in groups:
    g.config = EnvConfig(episode_steps=10)
hb = HeteroBatch(groups, master_seed=1, policy_seed=2)
hb.reset()
for _ in range(12):
    hb.multi_random_step()
torch.cuda.synchronize()
print("multi", hb.multi_info())
hb.close()
# PPO at small batches: the one-kernel rollout (ragged CTAs) and the fused update
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

for B in (16, 37):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=7)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=6, use_graph=False, n_minibatches=2, update_epochs=1))
    tr.iterate()
    torch.cuda.synchronize()
    print("ppo", B, tr._fused_rollout, tr._fused_update, env.last_step_mode())
    env.close()
print("ok")
