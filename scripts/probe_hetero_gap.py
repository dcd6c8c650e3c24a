"""Where the C5 heterogeneous step loses against homogeneous batches: each
station layout run as one homogeneous 2^20-env batch (random actions, whole
day), then as a 12-group hetero batch of that layout only, then the full
36-group sweep."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups  # noqa: E402

B = 1 << 20


def day_ms(step):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(288):
        step()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 288


groups = sweep_groups(B)
tot = 0.0
for li in range(3):
    g = groups[li]
    env = BatchEnv(g.config, g.station, g.dataset, batch_size=B)
    pol = DeviceRandomPolicy(0, env.n_ports, g.config.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    ms = day_ms(lambda: env.step(pol.actions(env), collect_infos=False))
    tot += ms / 3
    print(f"homogeneous {g.name.split('/')[-1]:17s}: {ms:.4f} ms/step  mode {env.last_step_mode()}")
    env.close()
    sub = [x for i, x in enumerate(sweep_groups(3 * B)) if i % 3 == li]
    hb = HeteroBatch(sub, master_seed=0, policy_seed=0)
    hb.reset()
    ms = day_ms(hb.graph_random_step)
    print(f"   12 groups of it ({hb.total} envs): {ms:.4f} ms/step  ({ms * B / hb.total:.4f} per 2^20)")
    hb.close()
print(f"homogeneous mix (1/3 each): {tot:.4f} ms/step per 2^20 envs  {B / tot * 1e3:.3e}")
for lf in (False, True):
    hb = HeteroBatch(groups, master_seed=0, policy_seed=0, longest_first=lf)
    hb.reset()
    ms = day_ms(hb.graph_random_step)
    print(f"36-group sweep (longest_first={lf}): {ms:.4f} ms/step  {B / ms * 1e3:.3e}")
    hb.close()
