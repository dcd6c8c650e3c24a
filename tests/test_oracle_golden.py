"""Pin the CPU oracle: it must replay the reference's golden trajectories bit for bit.

The fixtures were produced by the reference implementation itself
(scripts/make_golden.py); the oracle is driven with the fixture's recorded
actions and must reproduce every output exactly (assert_array_equal, the
reference's own parity standard, tests/test_backend_parity.py:61-71).
"""

import numpy as np
import pytest

from oracle.harness import HostBatch, HostRandomPolicy, ref_available
from scenarios import NAMES, Fixture

OUT_KEYS = ("breakdown", "flows", "declined", "arrivals_m", "dep_n", "term_overtime", "i_att", "i_used",
            "delivered", "b_delivered")
DEP_KEYS = ("dep_port", "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc")


def replay(fx: Fixture, core: str):
    hb = HostBatch(fx.tables(), fx.B, master_seed=fx.master_seed, core=core)
    obs0 = hb.reset()
    np.testing.assert_array_equal(obs0, fx["obs0"])
    acts = fx["actions"]
    for t in range(fx.steps):
        obs, r, d = hb.step(acts[t])
        np.testing.assert_array_equal(obs, fx["obs"][t], err_msg=f"obs t={t}")
        np.testing.assert_array_equal(r, fx["reward"][t], err_msg=f"reward t={t}")
        np.testing.assert_array_equal(d.astype(np.int8), fx["done"][t])
        o = hb.outs
        for k in OUT_KEYS:
            np.testing.assert_array_equal(getattr(o, k), fx[k][t], err_msg=f"{k} t={t}")
        dn = o.dep_n
        for k in DEP_KEYS:
            got = np.where(np.arange(fx.station.n_ports)[None, :] < dn[:, None], getattr(o, k), 0)
            np.testing.assert_array_equal(got, fx[k][t], err_msg=f"{k} t={t}")
        np.testing.assert_array_equal(np.where(d[:, None], o.ep_stats, 0.0), fx["ep_stats"][t])
        np.testing.assert_array_equal(hb.states.step, fx["step"][t])
        np.testing.assert_array_equal(hb.states.day, fx["day"][t])
        np.testing.assert_array_equal(hb.states.episode, fx["episode"][t])
    s = hb.states
    for k in ("occ", "i_drawn", "soc", "de", "dtrem", "cap", "rbar", "tau", "pref", "rhat", "b_i", "b_soc",
              "b_rhat", "env_seed", "ep_profit", "ep_reward", "ep_missing", "ep_energy", "ep_overtime",
              "ep_declined", "ep_departures"):
        np.testing.assert_array_equal(getattr(s, k), fx[f"final_{k}"], err_msg=k)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_replays_reference_golden(name):
    replay(Fixture(name), "oracle")


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference kernel) not built")
@pytest.mark.parametrize("name", ["bp_battery_penalties", "c4_highway64", "parking_order"])
def test_ref_kernel_replays_golden(name):
    """The reference's own compiled kernel, driven by our harness, reproduces the fixtures too."""
    replay(Fixture(name), "ref")


def test_oracle_random_policy_matches_reference_actions():
    fx = Fixture("c1_default")
    pol = HostRandomPolicy(seed=fx.meta["policy_seed"], n_ports=16, k=10, rows=range(fx.B))
    for t in range(5):
        np.testing.assert_array_equal(pol.actions(), fx["actions"][t])


def test_oracle_thread_count_invariant():
    fx = Fixture("c1_default")
    res = []
    for threads in (1, 4):
        hb = HostBatch(fx.tables(), fx.B, master_seed=fx.master_seed, threads=threads)
        hb.reset()
        hb.core.threads = threads
        for t in range(40):
            obs, r, d = hb.step(fx["actions"][t])
        res.append((obs, r))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
