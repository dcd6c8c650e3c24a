"""Single vy_step at small batches: tile kernel vs the one-warp-per-env kernel
(staged uint8 actions, auto-reset), CUDA-graph replay of 50 steps, us per step.
python scripts/probe_step_small.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup()
for B in (16, 256, 1024, 4096, 8192):
    res = {}
    for wide in (0, 1):
        env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
        env.set_wide(wide)
        pol = DeviceRandomPolicy(0, env.n_ports, rc.env.discretization_k)
        pol.bind(range(B))
        env.reset(as_numpy=False)
        acts = torch.stack([pol.actions(env).clone() for _ in range(50)])
        for t in range(120):  # into the day
            env.step(acts[t % 50], collect_infos=False)
        env.step(acts[0], collect_infos=False)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for t in range(50):
                env.step(acts[t], collect_infos=False)
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(4):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        res[wide] = s.elapsed_time(e) / 200 * 1e3
        env.close()
    print(f"B={B:5d} tile {res[0]:7.2f} us/step  wide {res[1]:7.2f} us/step", flush=True)
