"""The small-batch rollout (k_rollout_wide: one warp per env, one lane per
port, the reference's sequential sums done in port order with warp shuffles)
against the reference itself (golden fixture c1_default: config C1, 16 envs x
300 steps of the reference's RandomPolicy) and against the one-thread-per-env
rollout (bit for bit: obs, reward, done every step and the final state) on the
default station, a nested-splitter tree (Spec<2>, frequent rescales) and an
8-port station, across episode boundaries."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from scenarios import Fixture  # noqa: E402

STATE_KEYS = ("occ", "soc", "de", "i_drawn", "dtrem", "pref", "step", "day", "episode", "ep_reward", "ep_profit",
              "ep_missing", "ep_energy", "ep_overtime", "ep_declined", "ep_departures")


def _rollout(env, T, seed, call0=0):
    B = env.batch_size
    obs = torch.empty(T, B, env.obs_length, device="cuda")
    rew = torch.empty(T, B, device="cuda")
    done = torch.empty(T, B, dtype=torch.uint8, device="cuda")
    env.rollout(T, seed, call0, obs, rew, done)
    return obs, rew, done


def test_wide_rollout_reproduces_the_reference_c1():
    from paper_2507_01522_b200.batch import BatchEnv

    fx = Fixture("c1_default")
    env = BatchEnv(fx.config, fx.station, fx.dataset, batch_size=fx.B, master_seed=fx.master_seed)
    env.set_wide(1)
    obs0 = env.reset(as_numpy=False)
    np.testing.assert_array_equal(obs0.cpu().numpy(), fx["obs0"].astype(np.float32))
    obs, rew, done = _rollout(env, fx.steps, fx.meta["policy_seed"])
    assert env.last_step_mode() == 11  # the wide rollout ran
    np.testing.assert_array_equal(obs.cpu().numpy(), fx["obs"].astype(np.float32))
    np.testing.assert_array_equal(rew.cpu().numpy(), fx["reward"].astype(np.float32))
    np.testing.assert_array_equal(done.cpu().numpy(), fx["done"].astype(np.uint8))
    st = env.reference_state()
    for k in ("occ", "soc", "de", "i_drawn", "dtrem", "pref", "step", "day", "episode", "ep_profit", "ep_reward",
              "ep_missing", "ep_energy", "ep_overtime", "ep_declined", "ep_departures"):
        np.testing.assert_array_equal(st[k], fx[f"final_{k}"], err_msg=k)
    env.close()


def _setup(kind):
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.exogenous import generate_synthetic_defaults
    from paper_2507_01522_b200.station import preset_station

    if kind == "default":
        rc = default_setup(EnvConfig(episode_steps=120), days=30)
        return rc.env, rc.station, rc.dataset, 11
    if kind == "nested":
        return (EnvConfig(episode_steps=100), preset_station("nested_splitters", 4, 12),
                generate_synthetic_defaults("highway", "high", "eu", seed=0, days=30), 12)
    return (EnvConfig(episode_steps=90), preset_station("single_type", 0, 8),
            generate_synthetic_defaults("work", "high", "us", seed=0, days=30), 11)


@pytest.mark.parametrize("kind,B", [("default", 1000), ("default", 33), ("nested", 700), ("single", 500)])
def test_wide_rollout_equals_tile_rollout(kind, B):
    from paper_2507_01522_b200.batch import BatchEnv

    cfg, st, ds, mode = _setup(kind)
    envs = [BatchEnv(cfg, st, ds, batch_size=B, master_seed=7) for _ in range(2)]
    envs[0].set_wide(0)
    envs[1].set_wide(1)
    for e in envs:
        e.reset(as_numpy=False)
    T1, T2 = 130, 110  # two launches (state carried over), past the episode ends
    out = []
    for e in envs:
        r1 = _rollout(e, T1, 5, 0)
        r2 = _rollout(e, T2, 5, T1)
        out.append([torch.cat([a, b_]) for a, b_ in zip(r1, r2)])
    assert envs[1].last_step_mode() == mode
    for name, a, b_ in zip(("obs", "reward", "done"), out[0], out[1]):
        torch.testing.assert_close(b_, a, rtol=0, atol=0, msg=name)
    s0, s1 = envs[0].reference_state(), envs[1].reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(s1[k], s0[k], err_msg=k)
    for e in envs:
        e.close()


@pytest.mark.parametrize("kind,B", [("default", 1024), ("nested", 96)])
def test_wide_single_step_equals_tile_step(kind, B):
    """vy_step with staged uint8 actions (the PPO rollout's call) on the
    one-warp-per-env kernel == the tile kernel, step by step; an out-of-range
    action is clamped and flagged the same way."""
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    cfg, st, ds, mode = _setup(kind)
    envs = [BatchEnv(cfg, st, ds, batch_size=B, master_seed=9) for _ in range(2)]
    envs[0].set_wide(0)
    envs[1].set_wide(1)
    pol = DeviceRandomPolicy(4, envs[0].n_ports, cfg.discretization_k)
    pol.bind(range(B))
    for e in envs:
        e.reset(as_numpy=False)
    for t in range(cfg.episode_steps + 15):
        a = pol.actions(envs[0]).clone()
        outs = [e.step(a, collect_infos=False)[:3] for e in envs]
        assert envs[1].last_step_mode() == mode and envs[0].last_step_mode() in (1, 2)
        for name, x, y in zip(("obs", "reward", "done"), outs[0], outs[1]):
            torch.testing.assert_close(y, x, rtol=0, atol=0, msg=f"{name} t={t}")
    s0, s1 = envs[0].reference_state(), envs[1].reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(s1[k], s0[k], err_msg=k)
    bad = pol.actions(envs[1]).clone()
    bad[3, 1] = 2 * cfg.discretization_k + 5
    for e in envs:
        e.step(bad, collect_infos=False)
    with pytest.raises(ValueError):
        envs[1].check_errors()
    for e in envs:
        e.close()
