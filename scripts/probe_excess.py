"""How often the capacity-tree rescale runs (excess > 0) per layout: the
info block's c_constraint column over one day, random actions, 2^16 envs."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import EnvConfig, _native as nat  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.exogenous import generate_synthetic_defaults  # noqa: E402
from paper_2507_01522_b200.hetero import _LAYOUTS  # noqa: E402
from paper_2507_01522_b200.station import preset_station  # noqa: E402

B = 1 << 16
cfg = EnvConfig()
ds = generate_synthetic_defaults("shopping", "medium", "eu", seed=0, days=365)
for layout, ac, dc in _LAYOUTS:
    env = BatchEnv(cfg, preset_station(layout, ac, dc), ds, batch_size=B)
    env.outs.ensure_info()
    env._bind()
    pol = DeviceRandomPolicy(0, env.n_ports, cfg.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    hits = torch.zeros((), device="cuda")
    warp_hits = torch.zeros((), device="cuda")
    for _ in range(288):
        a = pol.actions(env)
        nat.check(env._lib.vy_step(env._h, a.data_ptr(), 0, env.n_ports + 1, 1, nat.F_AUTO_RESET | nat.F_INFOS,
                                   None, env._stream), "step")
        ex = env.outs.info["breakdown"][1, :B] > 0
        hits += ex.float().mean()
        warp_hits += ex.view(-1, 32).any(dim=1).float().mean()
    print(f"{layout:18s} nodes {env.tables.n_nodes:2d}: rescale in {hits.item() / 288 * 100:.2f}% of env-steps, "
          f"{warp_hits.item() / 288 * 100:.1f}% of warp-steps")
    env.close()
