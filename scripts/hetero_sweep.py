import sys
sys.path.insert(0, ".")
import torch
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups
B = 1 << 20
for tpw in (2, 3, 4):
    for ns in (9, 12, 18, 24):
        hb = HeteroBatch(sweep_groups(B), master_seed=0, policy_seed=0, n_streams=ns, tiles_per_warp=tpw)
        hb.reset()
        for _ in range(3):
            hb.graph_random_step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(288):
            hb.graph_random_step()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 288
        print(f"tpw {tpw} streams {ns:3d}: {ms:.4f} ms/step {B / ms * 1e3:.3e}")
        hb.close()
