"""Heterogeneous C5 step (36 config groups, one CUDA graph per step): ms per
step over a whole day vs the number of streams the groups are spread over."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups  # noqa: E402

B = 1 << 20
for ns in [int(x) for x in (sys.argv[1:] or ["4", "8", "12", "18", "36"])]:
    hb = HeteroBatch(sweep_groups(B), master_seed=0, policy_seed=0, n_streams=ns)
    hb.reset()
    for _ in range(3):
        hb.graph_random_step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(288):
        hb.graph_random_step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 288
    print(f"streams {ns:3d}: {ms:.4f} ms/step  {B / ms * 1e3:.3e} env-steps/s")
    hb.close()
