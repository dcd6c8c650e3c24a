"""Minibatch row gather of the PPO update (307k of 1.23M rows, 112 bf16
each): advanced indexing vs index_select."""
import torch

n, w, mb = 1228800, 112, 307200
obs = torch.randn(n, w, device="cuda").to(torch.bfloat16)
idx = torch.randperm(n, device="cuda")[:mb]
act = torch.randint(0, 21, (n, 17), device="cuda", dtype=torch.uint8)
import sys
sys.path.insert(0, ".")
from paper_2507_01522_b200.ppo import gather_rows  # noqa: E402
fns = {"vy_gather_rows": lambda: gather_rows(obs, idx), "obs[idx]": lambda: obs[idx], "index_select": lambda: obs.index_select(0, idx),
       "act[idx]": lambda: act[idx], "act index_select": lambda: act.index_select(0, idx),
       "sorted idx obs[idx]": lambda: obs[idx.sort().values]}
for name, f in fns.items():
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:20s} {s.elapsed_time(e) / 20 * 1e3:8.1f} us")
