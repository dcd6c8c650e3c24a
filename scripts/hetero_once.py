import sys
sys.path.insert(0, ".")
import torch
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups
hb = HeteroBatch(sweep_groups(1 << 20), master_seed=0, policy_seed=0, n_streams=16)
hb.reset()
for _ in range(140):
    hb.random_step()
torch.cuda.synchronize()
