"""Heterogeneous batch in ONE launch (config C5, k_step_multi): every group's
obs / reward / done and final state equal the per-group launches bit for bit
(which tests/test_gpu_hetero.py pins to standalone BatchEnvs and the CPU
oracle), eagerly and replayed from a CUDA graph, across episode boundaries
and with a ragged last group."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

STATE = ("occ", "soc", "de", "i_drawn", "dtrem", "episode", "day", "ep_reward", "ep_profit")


def _pair(groups, episode_steps):
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.hetero import HeteroBatch

    for g in groups:
        g.config = EnvConfig(episode_steps=episode_steps)
    a = HeteroBatch(groups, master_seed=3, policy_seed=5)
    b = HeteroBatch(groups, master_seed=3, policy_seed=5)
    a.reset()
    b.reset()
    return a, b


def _same(a, b, states=False):
    for ea, eb in zip(a.envs, b.envs):
        torch.testing.assert_close(eb.outs.obs, ea.outs.obs, rtol=0, atol=0)
        torch.testing.assert_close(eb.outs.reward, ea.outs.reward, rtol=0, atol=0)
        torch.testing.assert_close(eb.outs.done, ea.outs.done, rtol=0, atol=0)
        if states:
            sa, sb = ea.reference_state(), eb.reference_state()
            for k in STATE:
                np.testing.assert_array_equal(sb[k], sa[k], err_msg=k)


def test_multi_launch_equals_group_launches_c5_sweep():
    from paper_2507_01522_b200.hetero import sweep_groups

    groups = sweep_groups(total_envs=36 * 96 + 45, days=20)  # all 36 groups, ragged last one
    a, b = _pair(groups, episode_steps=40)
    info = b.multi_info()
    # nested splitters force the any-tree path; 3 regional car catalogues x 3 station layouts
    assert info["mode"] == 2 and info["profile_sets"] == 3 and info["station_sets"] == 3, info
    for t in range(90):
        a.random_step()
        b.multi_random_step()
        if t % 11 == 0 or t in (38, 39, 40, 41):
            _same(a, b)
    _same(a, b, states=True)
    a.close()
    b.close()


def test_multi_launch_fast_tree_groups_and_graph_replay():
    from paper_2507_01522_b200.hetero import sweep_groups

    groups = [g for i, g in enumerate(sweep_groups(total_envs=36 * 64, days=20)) if i % 3 != 2][:10]
    a, b = _pair(groups, episode_steps=25)
    assert b.multi_info()["mode"] == 1  # single / multi_type stations: <= 4 tree nodes
    for t in range(60):
        a.random_step()
        b.graph_multi_step()
        if t % 7 == 0 or t in (23, 24, 25):
            _same(a, b)
    _same(a, b, states=True)
    a.close()
    b.close()
