"""k_step day-average time for each station layout of the C5 sweep run
homogeneously (2^20 envs, shopping/medium/eu, random actions)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import EnvConfig  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.exogenous import generate_synthetic_defaults  # noqa: E402
from paper_2507_01522_b200.hetero import _LAYOUTS  # noqa: E402
from paper_2507_01522_b200.station import preset_station  # noqa: E402

B = 1 << 20
cfg = EnvConfig()
for scen, traffic in (("shopping", "medium"), ("highway", "high")):
    ds = generate_synthetic_defaults(scen, traffic, "eu", seed=0, days=365)
    for layout, ac, dc in _LAYOUTS:
        env = BatchEnv(cfg, preset_station(layout, ac, dc), ds, batch_size=B)
        pol = DeviceRandomPolicy(0, env.n_ports, cfg.discretization_k)
        pol.bind(range(B))
        env.reset(as_numpy=False)
        for _ in range(5):
            env.step(pol.actions(env), collect_infos=False)
        ev = []
        for _ in range(288):
            a = pol.actions(env)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            env.step(a, collect_infos=False)
            e.record()
            ev.append((s, e))
        torch.cuda.synchronize()
        ms = sum(s.elapsed_time(e) for s, e in ev) / len(ev)
        print(f"{scen}/{traffic} {layout:18s} ports {env.n_ports:2d} nodes {env.tables.n_nodes:2d}: "
              f"k_step {ms:.4f} ms  ({B / ms * 1e3:.3e} env-steps/s)")
        env.close()
