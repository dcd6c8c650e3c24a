"""Fused RandomPolicy step (vy_step_random) == RandomPolicy.actions + step.

The throughput_probe loop body `env.step(policy.actions(obs))`
(engine.py:541-545, policies.py:51-73) as one kernel must be bit-identical to
the two-launch form, to the reference's actions (golden fixture c1_default)
and to the CPU oracle.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.harness import HostBatch, HostRandomPolicy  # noqa: E402
from scenarios import Fixture  # noqa: E402

STATE = ("occ", "soc", "de", "i_drawn", "dtrem", "step", "day", "episode", "ep_reward", "ep_profit")


def _pair(B, obs_dtype, steps, device_counter=False, seed=7, index0=0, master=3, rc=None):
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = rc or default_setup(EnvConfig(episode_steps=40), days=20)
    envs = [BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=master, obs_dtype=obs_dtype)
            for _ in range(2)]
    pols = [DeviceRandomPolicy(seed, envs[0].n_ports, rc.env.discretization_k) for _ in range(2)]
    for p in pols:
        p.bind(range(index0, index0 + B))
    for e in envs:
        e.reset(as_numpy=False)
    for t in range(steps):
        a = pols[0].actions(envs[0]).clone()
        o0, r0, d0, _ = envs[0].step(a, collect_infos=False)
        o1, r1, d1, _ = envs[1].step_random(pols[1], keep_actions=True, device_counter=device_counter)
        np.testing.assert_array_equal(pols[1].last_actions.cpu().numpy(), a.cpu().numpy(), err_msg=f"a t={t}")
        np.testing.assert_array_equal(o1.cpu().numpy(), o0.cpu().numpy(), err_msg=f"obs t={t}")
        np.testing.assert_array_equal(r1.cpu().numpy(), r0.cpu().numpy(), err_msg=f"reward t={t}")
        np.testing.assert_array_equal(d1.cpu().numpy(), d0.cpu().numpy(), err_msg=f"done t={t}")
    s0, s1 = envs[0].reference_state(), envs[1].reference_state()
    for k in STATE:
        np.testing.assert_array_equal(s1[k], s0[k], err_msg=k)
    modes = [e.last_step_mode() for e in envs]
    for e in envs:
        e.check_errors()
        e.close()
    return modes


@pytest.mark.parametrize("B", [4096, 1000, 33])
def test_fused_policy_step_equals_two_launches_lean(B):
    modes = _pair(B, torch.float32, 90)  # 90 steps: two auto-resets at episode_steps = 40
    if B % 32 == 0:
        assert modes == [1, 1]


def test_fused_policy_step_generic_f64():
    assert _pair(256, torch.float64, 50, index0=1000)[1] == 0


def test_fused_policy_step_device_counter():
    _pair(512, torch.float32, 45, device_counter=True)


def test_fused_policy_step_graph_replay():
    """One captured vy_step_random replayed T times == T eager steps."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = default_setup()
    B, T = 2048, 30
    envs = [BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=5) for _ in range(2)]
    pols = [DeviceRandomPolicy(2, 16, 10) for _ in range(2)]
    for p in pols:
        p.bind(range(B))
    for e in envs:
        e.reset(as_numpy=False)
    for _ in range(T):
        envs[0].step_random(pols[0])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        envs[1].step_random(pols[1], device_counter=True)  # warm-up replay = call 0
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            envs[1].step_random(pols[1], device_counter=True)
    for _ in range(T - 1):
        g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(envs[1].outs.obs.cpu().numpy(), envs[0].outs.obs.cpu().numpy())
    s0, s1 = envs[0].reference_state(), envs[1].reference_state()
    for k in STATE:
        np.testing.assert_array_equal(s1[k], s0[k], err_msg=k)
    for e in envs:
        e.close()


def test_fused_policy_step_equals_reference_actions_and_oracle():
    """c1_default: the fused step's actions are the reference's RandomPolicy
    rows, and its trajectory equals the CPU oracle's."""
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    fx = Fixture("c1_default")
    env = BatchEnv(fx.config, fx.station, fx.dataset, batch_size=fx.B, master_seed=fx.master_seed,
                   obs_dtype=torch.float64)
    pol = DeviceRandomPolicy(fx.meta["policy_seed"], 16, 10)
    pol.bind(range(fx.B))
    np.testing.assert_array_equal(env.reset(as_numpy=False).cpu().numpy(), fx["obs0"])
    for t in range(fx.steps):
        obs, r, d, _ = env.step_random(pol, keep_actions=True)
        np.testing.assert_array_equal(pol.last_actions.cpu().numpy(), fx["actions"][t], err_msg=f"a t={t}")
        np.testing.assert_array_equal(obs.cpu().numpy(), fx["obs"][t], err_msg=f"obs t={t}")
        np.testing.assert_array_equal(r.cpu().numpy(), fx["reward"][t])
    env.close()

    # fresh seeds at 2^14 envs against the multi-threaded oracle
    from paper_2507_01522_b200 import default_setup

    rc = default_setup()
    B = 1 << 14
    from paper_2507_01522_b200.streams import vstream_key

    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=11, global_offset=B)
    ref = HostBatch(env.tables, B, env_seeds=vstream_key(11, np.arange(B, 2 * B, dtype=np.int64)), threads=8)
    pol = DeviceRandomPolicy(9, 16, 10)
    pol.bind(range(B, 2 * B))
    hpol = HostRandomPolicy(9, 16, 10, range(B, 2 * B), threads=8)
    env.reset(as_numpy=False)
    ref.reset()
    for t in range(60):
        obs, r, d, _ = env.step_random(pol)
        obs_h, r_h, d_h = ref.step(hpol.actions())
        np.testing.assert_array_equal(obs.cpu().numpy(), obs_h.astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(r.cpu().numpy(), r_h.astype(np.float32))
        np.testing.assert_array_equal(d.cpu().numpy().astype(bool), d_h)
    env.close()


@pytest.mark.parametrize("B", [1000, 4096])
def test_fused_policy_step_streamed_c4_tile(B):
    """Config C4's 64-port battery station runs the streamed tile (Spec<4>:
    currents resident, soc / energy / dwell read a few ports ahead, obs
    through the per-port chunk ring).  It equals the two-launch form — the
    generic kernel for the ragged B = 1000, the same streamed kernel fed
    staged actions for B = 4096 — over an episode boundary (auto-reset obs)."""
    from paper_2507_01522_b200 import EnvConfig, RunConfig
    from paper_2507_01522_b200.workloads import c4_setup

    c4 = c4_setup(days=20)
    env = EnvConfig(battery_enabled=True, alpha=c4.env.alpha, beta=c4.env.beta, episode_steps=30)
    rc = RunConfig(env=env, station=c4.station, dataset=c4.dataset)
    modes = _pair(B, torch.float32, 70, rc=rc)
    assert modes[1] == 4 and modes[0] == (0 if B % 32 else 4), modes

