"""The reference-facing numpy path: BatchEnv.step(np.int64 actions) -> numpy
float64 obs / rewards / dones (the exact drop-in), timed per step on the host."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402

rc = default_setup()
print("torch threads", torch.get_num_threads())
for B in (1 << 16, 1 << 20):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, obs_dtype=torch.float64)
    env.reset()
    rng = np.random.default_rng(0)
    acts = rng.integers(0, 21, size=(B, 17), dtype=np.int64)
    for _ in range(4):  # the caller keeps the last step's arrays: warms a 2-deep output ring
        obs, r, d, _ = env.step(acts, collect_infos=False)
    n = 10
    t0 = time.perf_counter()
    for _ in range(n):
        obs, r, d, _ = env.step(acts, collect_infos=False)
    dt = (time.perf_counter() - t0) / n
    print(f"B={B}: {dt * 1e3:.1f} ms/step  {B / dt:.3e} env-steps/s  obs {obs.dtype} {obs.shape}")
    t0 = time.perf_counter()
    for _ in range(n):
        env._device_actions(acts)
    torch.cuda.synchronize()
    ta = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        pins = [env._pinned(k, t) for k, t in (("obs", env.outs.obs), ("rew", env.outs.reward))]
        torch.cuda.synchronize()
    td = (time.perf_counter() - t0) / n
    from paper_2507_01522_b200.batch import _fresh
    t0 = time.perf_counter()
    for _ in range(n):
        _fresh(pins[0], torch.float64)
    th = (time.perf_counter() - t0) / n
    print(f"   actions {ta * 1e3:.1f} ms  d2h {td * 1e3:.1f} ms  host obs copy {th * 1e3:.1f} ms")
    env.close()
