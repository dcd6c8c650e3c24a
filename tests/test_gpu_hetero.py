"""Heterogeneous batches (config C5): each group equals a standalone BatchEnv
with the same global env indices, bit for bit, and the CPU oracle on a subset."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_hetero_groups_equal_standalone_envs_and_oracle():
    from oracle.harness import HostBatch, HostRandomPolicy
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy
    from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups
    from paper_2507_01522_b200.streams import split_seed

    groups = sweep_groups(total_envs=36 * 40, days=20)[::9]  # 4 diverse groups
    for g in groups:
        g.config = EnvConfig(episode_steps=30)
    hb = HeteroBatch(groups, master_seed=3, policy_seed=5)
    obs = [o.clone() for o in hb.reset()]
    frames = [[o] for o in obs]
    for _ in range(45):
        for gi, (o, r, d) in enumerate(hb.random_step()):
            frames[gi].append(o.clone())
    off = 0
    for gi, g in enumerate(groups):
        env = BatchEnv(g.config, g.station, g.dataset, batch_size=g.batch_size, master_seed=3, global_offset=off)
        pol = DeviceRandomPolicy(5, env.n_ports, 10)
        pol.bind(range(off, off + g.batch_size))
        ref = [env.reset(as_numpy=False).clone()]
        for _ in range(45):
            o, r, d, _ = env.step(pol.actions(env), collect_infos=False)
            ref.append(o.clone())
        torch.testing.assert_close(torch.stack(frames[gi]), torch.stack(ref), rtol=0, atol=0)
        # oracle on three rows of this group
        rows = [0, g.batch_size // 2, g.batch_size - 1]
        h = HostBatch(env.tables, len(rows), env_seeds=[split_seed(3, off + i) for i in rows])
        hp = HostRandomPolicy(5, env.n_ports, 10, [off + i for i in rows])
        want = [h.reset()]
        for _ in range(45):
            want.append(h.step(hp.actions())[0])
        got = torch.stack(frames[gi])[:, rows].cpu().numpy()
        np.testing.assert_array_equal(got, np.array(want).astype(np.float32))
        env.close()
        off += g.batch_size
    hb.close()


def test_graph_replayed_hetero_step_equals_eager():
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups

    groups = sweep_groups(total_envs=36 * 64, days=20)[::7]
    for g in groups:
        g.config = EnvConfig(episode_steps=20)
    a = HeteroBatch(groups, master_seed=1, policy_seed=2)
    b = HeteroBatch(groups, master_seed=1, policy_seed=2)
    a.reset()
    b.reset()
    for _ in range(33):  # crosses an auto-reset
        oa = [o.clone() for o, _, _ in a.random_step()]
        b.graph_random_step()
        ob = [e.outs.obs.clone() for e in b.envs]
        for x, y in zip(oa, ob):
            torch.testing.assert_close(x, y, rtol=0, atol=0)
    for ea, eb in zip(a.envs, b.envs):
        sa, sb = ea.reference_state(), eb.reference_state()
        for k in ("soc", "de", "occ", "step", "episode", "ep_reward"):
            np.testing.assert_array_equal(sa[k], sb[k])
    a.close()
    b.close()
