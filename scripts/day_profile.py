"""k_step time and station occupancy across one 288-step episode (bench workload)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

rc = default_setup()
B = 1 << 20
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
pol = DeviceRandomPolicy(0, 16, 10)
pol.bind(range(B))
env.reset(as_numpy=False)
out = []
for t in range(2 * 288):
    a = pol.actions(env)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    env.step(a, collect_infos=False)
    e.record()
    torch.cuda.synchronize()
    occ = float((env.states.port_meta[:, :B] & 1).float().mean()) if t % 8 == 0 else None
    out.append((t, s.elapsed_time(e), occ))
ms = [o[1] for o in out[288:]]
print("episode-2 mean ms", sum(ms) / len(ms), "min", min(ms), "max", max(ms))
for t, m, occ in out[288::8]:
    print(t - 288, round(m, 4), occ)
json.dump(out, open("gpurun_out/day_profile.json", "w"))
