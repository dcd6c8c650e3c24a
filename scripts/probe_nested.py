"""Day-average step time of one homogeneous 2^20-env batch per C5 station
layout (random actions), for A/B-ing tree-fitting variants."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.hetero import sweep_groups  # noqa: E402

B = 1 << 20
groups = sweep_groups(B)
res = []
for li in range(3):
    g = groups[li]
    env = BatchEnv(g.config, g.station, g.dataset, batch_size=B)
    pol = DeviceRandomPolicy(0, env.n_ports, g.config.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    for _ in range(3):
        env.step(pol.actions(env), collect_infos=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(288):
        env.step(pol.actions(env), collect_infos=False)
    e.record()
    torch.cuda.synchronize()
    res.append(f"{g.name.split('/')[-1]} {s.elapsed_time(e) / 288:.4f}")
    env.close()
print("  ".join(res))
