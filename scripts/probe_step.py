"""Micro-probe of k_step on the bench workload: full step vs memory-only (flag 0x200)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import _native as nat, default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup()
B = 1 << 20
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
pol = DeviceRandomPolicy(0, 16, 10)
pol.bind(range(B))
env.reset(as_numpy=False)
a = pol.actions(env)
for flags, name in ((1, "full"), (1 | 0x200, "memory-only (no transition math)"), (1 | 0x200 | 0x400, "memory-only, no obs stores"), (1 | 0x200 | 0x800, "memory-only, no state stores"), (1 | 0x200 | 0x400 | 0x800, "memory-only, loads only")):
    ts = []
    for i in range(25):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        nat.check(env._lib.vy_step(env._h, a.data_ptr(), 0, 17, 1, flags, None, env._stream), "step")
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts = sorted(ts[5:])
    print(name, "median ms", ts[len(ts) // 2], "eqGB/s", 1414 * B / (ts[len(ts) // 2] / 1e3) / 1e9)
