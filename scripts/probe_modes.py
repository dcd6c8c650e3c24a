"""k_step time of the default station in each output mode: lean float32
(throughput path) and exact float64 obs (the generic kernel, drop-in numpy
path).  (Infos mode is not timed here: BatchEnv.step then builds the
reference's per-env Python info dicts on the host.)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup()
B = 1 << 20
for name, dt, infos in (("f32 lean", torch.float32, False), ("f64 obs", torch.float64, False)):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, obs_dtype=dt)
    pol = DeviceRandomPolicy(0, env.n_ports, rc.env.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    for _ in range(5):
        env.step(pol.actions(env), collect_infos=infos)
    ev = []
    for _ in range(96):
        a = pol.actions(env)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        env.step(a, collect_infos=infos)
        e.record()
        ev.append((s, e))
        env.step(pol.actions(env), collect_infos=infos)
        env.step(pol.actions(env), collect_infos=infos)
    torch.cuda.synchronize()
    ms = sum(s.elapsed_time(e) for s, e in ev) / len(ev)
    print(f"{name:12s}: step {ms:.4f} ms  ({B / ms * 1e3:.3e} env-steps/s)")
    env.close()
