"""The one-kernel PPO rollout (vy_ppo_rollout: per CTA 16 envs x T steps of
tcgen05 policy pass + env step, then the bootstrap value) against the
per-step pair it replaces (vy_policy_step + the one-warp-per-env vy_step,
2T + 1 launches): same network, same sampler seed and counter, so every
rollout buffer (obs, actions, log-probabilities, values, rewards, dones),
the env state afterwards and the sampler counter must agree bit for bit —
on the default station, a nested-splitter tree (Spec<2>), an 8-port station,
ragged CTAs (B not a multiple of 16) and two rollouts in a row (state and
counter carried over).  The env side is also replayed on the CPU oracle by
test_gpu_ppo.py's rollout tests, which now run this kernel."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

STATE_KEYS = ("occ", "soc", "de", "i_drawn", "dtrem", "pref", "step", "day", "episode", "ep_reward", "ep_profit",
              "ep_missing", "ep_energy", "ep_overtime", "ep_declined", "ep_departures")
BUFFERS = ("obs", "actions", "logp", "values", "rewards", "dones")


def _setup(kind):
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.exogenous import generate_synthetic_defaults
    from paper_2507_01522_b200.station import preset_station

    if kind == "default":
        rc = default_setup(EnvConfig(episode_steps=40), days=30)
        return rc.env, rc.station, rc.dataset, 21
    if kind == "nested":
        return (EnvConfig(episode_steps=30), preset_station("nested_splitters", 4, 12),
                generate_synthetic_defaults("highway", "high", "eu", seed=0, days=30), 22)
    return (EnvConfig(episode_steps=25), preset_station("single_type", 0, 8),
            generate_synthetic_defaults("work", "high", "us", seed=0, days=30), 21)


@pytest.mark.parametrize("kind,B", [("default", 16), ("default", 37), ("nested", 48), ("single", 20),
                                    ("default", 300)])
def test_fused_rollout_equals_per_step_pair(kind, B):
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    cfg, st, ds, mode = _setup(kind)
    T = 50  # past an episode end (auto-reset inside the kernel)
    trs = []
    for fused in (False, True):
        env = BatchEnv(cfg, st, ds, batch_size=B, master_seed=3)
        trs.append(PPOTrainer(env, PPOConfig(rollout_steps=T, use_graph=False, fused_rollout=fused,
                                             total_timesteps=10 * T * B)))
    ref, fus = trs
    for p, q in zip(ref.net.parameters(), fus.net.parameters()):
        assert torch.equal(p, q)
    for it in range(2):
        for tr in trs:
            tr.rollout()
        assert fus.env.last_step_mode() == mode and fus._fused_rollout
        assert ref.env.last_step_mode() != mode
        for name in BUFFERS:
            a, b = getattr(ref, name), getattr(fus, name)
            assert torch.equal(a, b), f"{name} differs (rollout {it}): {(a != b).sum().item()} elements"
        assert torch.equal(ref._sample_ctr, fus._sample_ctr)
        assert ref.env._t == fus.env._t
        for tr in trs:
            tr.obs[0].copy_(tr.obs[T])
    s0, s1 = ref.env.reference_state(), fus.env.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(s1[k], s0[k], err_msg=k)
    for tr in trs:
        tr.env.close()


def test_fused_rollout_graph_replays_and_learns():
    """The captured form (pack_policy + one kernel per replay) continues the
    env across replays and the trainer's iterations stay finite."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup()
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=16, master_seed=1)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=300))
    assert "vy_ppo_rollout" in tr.describe_rollout()
    launches0 = env.launch_count()
    for _ in range(3):
        st = tr.iterate()
    assert all(torch.isfinite(v).all() for v in st.values())
    assert env.last_step_mode() == 21
    assert env._t == int(env.states.view("step")[0])
    # warm-up rollout + capture (not executed) + replays: one env-side launch per executed rollout
    assert env.launch_count() - launches0 <= 3
    env.close()


def test_fused_rollout_unsupported_station_falls_back():
    """A battery station is outside the kernel (lean, no battery): the trainer
    falls back to the per-step pair on the first rollout."""
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup(EnvConfig(battery_enabled=True, episode_steps=30), days=20)
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=32, master_seed=2)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=10, use_graph=False))
    tr.rollout()
    assert not tr._fused_rollout
    assert torch.isfinite(tr.values).all()
    env.close()
