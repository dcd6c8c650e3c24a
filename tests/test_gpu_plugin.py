"""The reference's own, unmodified BatchEnv driving the CUDA core.

``plugin.register`` adds backend "cuda" to the installed reference package
(baseline/_ref: `pip install --target baseline/_ref` of /root/reference/pkg);
the engine's validation, worker split, auto-reset loop and infos are the
reference's code, the stepping core is ``CudaSimCore``.  Checked against the
reference's compiled kernel on the six scenarios of its backend-parity test
(pkg/tests/test_backend_parity.py:23-71) with the same comparisons, plus every
state slot, every info record and a multi-worker engine.
"""

import numpy as np
import pytest

from ref_scenarios import import_reference

voltyard = import_reference()
pytestmark = pytest.mark.skipif(voltyard is None, reason="reference not installed in baseline/_ref")

STATE = ("occ", "i_drawn", "soc", "de", "dtrem", "cap", "rbar", "tau", "pref", "rhat", "b_i", "b_soc", "b_rhat",
         "step", "day", "episode", "env_seed", "ep_profit", "ep_reward", "ep_missing", "ep_energy", "ep_overtime",
         "ep_declined", "ep_departures")
OUTS = ("obs", "reward", "done", "breakdown", "flows", "declined", "arrivals_m", "dep_n", "dep_port", "dep_missing",
        "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc", "term_overtime", "ep_stats", "i_att",
        "i_used", "delivered", "b_delivered")


def test_register_adds_the_cuda_backend():
    from paper_2507_01522_b200 import plugin

    plugin.register(voltyard)
    from voltyard import backends, engine

    assert "cuda" in backends.available_backends()
    assert engine.resolve_backend("cuda") == "cuda" and engine.resolve_backend("compiled") == "compiled"
    with pytest.raises(ValueError):
        engine.resolve_backend("nope")


def _trajectory(cfg, station, ds, backend, steps, B=3, workers=1, infos=True):
    from voltyard.engine import BatchEnv
    from voltyard.policies import RandomPolicy

    env = BatchEnv(cfg, station, ds, batch_size=B, master_seed=17, backend=backend, workers=workers)
    pol = RandomPolicy(seed=23, n_ports=station.n_ports, k=cfg.discretization_k)
    pol.bind(range(B))
    obs = env.reset()
    rec = {"obs0": obs.copy(), "steps": []}
    for _ in range(steps):
        obs, r, d, inf = env.step(pol.actions(obs), collect_infos=infos)
        row = {"obs": obs.copy(), "reward": r.copy(), "done": d.copy()}
        if infos:
            row.update({k: getattr(env.outs, k).copy() for k in OUTS})
            row["infos"] = inf
        rec["steps"].append(row)
    rec["state"] = {k: getattr(env.states, k).copy() for k in STATE}
    env.close()
    return rec


def _assert_same(a, b):
    np.testing.assert_array_equal(a["obs0"], b["obs0"])
    for t, (x, y) in enumerate(zip(a["steps"], b["steps"])):
        for k in x:
            if k == "infos":
                assert len(x[k]) == len(y[k])
                for p, q in zip(x[k], y[k]):
                    for f in ("flows", "breakdown", "departures", "declined", "arrivals_sampled", "done", "episode",
                              "battery_delivered_kwh"):
                        assert getattr(p, f) == getattr(q, f), f"info {f} t={t}"
                    for f in ("currents_attempted_a", "currents_applied_a", "delivered_kwh"):
                        np.testing.assert_array_equal(getattr(p, f), getattr(q, f), err_msg=f"info {f} t={t}")
            else:
                np.testing.assert_array_equal(x[k], y[k], err_msg=f"{k} t={t}")
    for k in STATE:
        np.testing.assert_array_equal(a["state"][k], b["state"][k], err_msg=f"state {k}")


def _cases():
    from ref_scenarios import scenario_cases

    return list(scenario_cases())


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(6), ids=["default", "battery+penalties", "no-discharge", "nested-station",
                                                "coarse-dt", "random-tree"])
def test_reference_batchenv_on_cuda_core_equals_compiled(idx):
    """test_backend_parity.py's trajectories (2 episodes, 3 envs, RandomPolicy 23)
    with every output, info record and state slot: CUDA core == compiled core."""
    from paper_2507_01522_b200 import plugin

    plugin.register(voltyard)
    name, cfg, station, ds = _cases()[idx]
    steps = 2 * cfg.episode_steps
    ref = _trajectory(cfg, station, ds, "compiled", steps)
    got = _trajectory(cfg, station, ds, "cuda", steps)
    _assert_same(ref, got)


@pytest.mark.gpu
def test_worker_threads_gather_into_one_launch():
    """workers > 1: the engine's slices (engine.py:446-456) are gathered; the
    trajectory equals the single-worker compiled run (tests/test_engine.py:78-86)."""
    from paper_2507_01522_b200 import plugin

    plugin.register(voltyard)
    name, cfg, station, ds = _cases()[0]
    ref = _trajectory(cfg, station, ds, "compiled", 150, B=37)
    got = _trajectory(cfg, station, ds, "cuda", 150, B=37, workers=4)
    _assert_same(ref, got)


@pytest.mark.gpu
def test_outputs_mirror_mode_large_batch(monkeypatch):
    """VOLTYARD_CUDA_MIRROR=outputs (device-resident state, infos off): the
    reference engine at 4096 envs of the default station through the
    auto-reset equals the compiled core on obs / reward / done / episode."""
    from voltyard.config import EnvConfig
    from voltyard.data import generate_synthetic_defaults
    from voltyard.topology import preset_station

    from paper_2507_01522_b200 import plugin

    plugin.register(voltyard)
    cfg = EnvConfig(episode_steps=96)
    st = preset_station("multi_type", 6, 10)
    ds = generate_synthetic_defaults("shopping", "high", "eu", seed=0, days=30)
    ref = _trajectory(cfg, st, ds, "compiled", 110, B=4096, infos=False)
    monkeypatch.setenv("VOLTYARD_CUDA_MIRROR", "outputs")
    got = _trajectory(cfg, st, ds, "cuda", 110, B=4096, infos=False)
    np.testing.assert_array_equal(ref["obs0"], got["obs0"])
    for t, (x, y) in enumerate(zip(ref["steps"], got["steps"])):
        for k in ("obs", "reward", "done"):
            np.testing.assert_array_equal(x[k], y[k], err_msg=f"{k} t={t}")
    for k in ("step", "day", "episode"):
        np.testing.assert_array_equal(ref["state"][k], got["state"][k], err_msg=k)
