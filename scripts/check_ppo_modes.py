"""PPO trainer in its non-default modes (torch head, eager rollout/update): three iterations each, finite stats."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_01522_b200 import default_setup
from paper_2507_01522_b200.batch import BatchEnv
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer
rc = default_setup()
for fused, graph in ((False, True), (False, False), (True, False)):
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=256, master_seed=1)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=20, fused_head=fused, use_graph=graph))
    for _ in range(3):
        st = tr.iterate()
    print(fused, graph, {k: round(float(v), 4) for k, v in st.items()})
    env.close()
