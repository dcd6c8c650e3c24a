"""CUDA step vs the reference: golden fixtures and the CPU oracle, bit for bit.

Bar (north_star): discrete state bit-exact, floats within rel 1e-5.  The
kernels reproduce the reference's float64 arithmetic exactly, so every check
here is assert_array_equal — float64 outputs equal the reference's values,
float32 outputs equal float32(reference).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.harness import HostBatch, HostRandomPolicy  # noqa: E402
from scenarios import NAMES, Fixture  # noqa: E402

OUT_KEYS = ("breakdown", "flows", "declined", "arrivals_m", "dep_n", "term_overtime", "i_att", "i_used",
            "delivered", "b_delivered")
DEP_KEYS = ("dep_port", "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc")
STATE_KEYS = ("occ", "i_drawn", "soc", "de", "dtrem", "cap", "rbar", "tau", "pref", "rhat", "b_i", "b_soc",
              "b_rhat", "step", "day", "episode", "env_seed", "ep_profit", "ep_reward", "ep_missing", "ep_energy",
              "ep_overtime", "ep_declined", "ep_departures")


def make_env(fx, **kw):
    from paper_2507_01522_b200.batch import BatchEnv

    return BatchEnv(fx.config, fx.station, fx.dataset, batch_size=fx.B, master_seed=fx.master_seed, **kw)


@pytest.mark.parametrize("name", NAMES)
def test_golden_trajectory_f64_with_infos(name):
    """Numpy drop-in path, float64 outputs, infos on: every output equals the reference's."""
    fx = Fixture(name)
    env = make_env(fx, obs_dtype=torch.float64)
    np.testing.assert_array_equal(env.reset(), fx["obs0"])
    for t in range(fx.steps):
        obs, r, d, infos = env.step(fx["actions"][t], collect_infos=True)
        np.testing.assert_array_equal(obs, fx["obs"][t], err_msg=f"obs t={t}")
        np.testing.assert_array_equal(r, fx["reward"][t], err_msg=f"reward t={t}")
        np.testing.assert_array_equal(d.astype(np.int8), fx["done"][t])
        o = env.reference_outputs()
        for k in OUT_KEYS:
            np.testing.assert_array_equal(o[k], fx[k][t], err_msg=f"{k} t={t}")
        dn = o["dep_n"]
        for k in DEP_KEYS:
            got = np.where(np.arange(fx.station.n_ports)[None, :] < dn[:, None], o[k], 0)
            np.testing.assert_array_equal(got, fx[k][t], err_msg=f"{k} t={t}")
        np.testing.assert_array_equal(np.where(d[:, None], o["ep_stats"], 0.0), fx["ep_stats"][t])
        assert len(infos) == fx.B and all(info.done == bool(x) for info, x in zip(infos, d))
    st = env.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(st[k], fx[f"final_{k}"], err_msg=k)
    env.close()


@pytest.mark.parametrize("name", ["c1_default", "c4_highway64", "bp_nested", "default_maxcharge"])
def test_golden_trajectory_f32_device_path(name):
    """Torch device path, float32 outputs, infos off: obs == float32(reference obs)."""
    fx = Fixture(name)
    env = make_env(fx)
    obs = env.reset(as_numpy=False)
    np.testing.assert_array_equal(obs.cpu().numpy(), fx["obs0"].astype(np.float32))
    acts = torch.as_tensor(fx["actions"], device="cuda")
    for t in range(fx.steps):
        obs, r, d, _ = env.step(acts[t], collect_infos=False)
        np.testing.assert_array_equal(obs.cpu().numpy(), fx["obs"][t].astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(r.cpu().numpy(), fx["reward"][t].astype(np.float32))
        np.testing.assert_array_equal(d.cpu().numpy(), fx["done"][t].astype(np.uint8))
    st = env.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(st[k], fx[f"final_{k}"], err_msg=k)
    env.check_errors()
    env.close()


LEAN = {"bp_coarse_dt": 1, "bp_default": 1, "bp_no_discharge": 1, "c1_default": 1, "default_maxcharge": 1,
        "bp_random_tree": 2, "c4_highway64": 4, "c5_nested_residential_us": 2, "c5_single_highway_world": 1,
        "c2_default_tile": 1}


@pytest.mark.parametrize("name", sorted(LEAN))
def test_golden_trajectory_lean_kernel(name):
    """The lean step instantiations (vy_device.cuh Spec<1> / <2> / <3>) need
    staged uint8 actions for whole 32-env tiles: the fixture's envs are rows
    0..B-1 of a 32-env batch (same seeds), extra rows get the fixture's first
    row of actions; rows 0..B-1 must reproduce the reference bit for bit."""
    fx = Fixture(name)
    from paper_2507_01522_b200.batch import BatchEnv

    env = BatchEnv(fx.config, fx.station, fx.dataset, batch_size=32, master_seed=fx.master_seed)
    obs = env.reset(as_numpy=False)
    np.testing.assert_array_equal(obs[: fx.B].cpu().numpy(), fx["obs0"].astype(np.float32))
    acts = np.repeat(fx["actions"][:, :1, :], 32, axis=1)
    acts[:, : fx.B] = fx["actions"]
    acts = torch.as_tensor(acts.astype(np.uint8), device="cuda")
    for t in range(fx.steps):
        obs, r, d, _ = env.step(acts[t], collect_infos=False)
        assert env.last_step_mode() == LEAN[name]
        np.testing.assert_array_equal(obs[: fx.B].cpu().numpy(), fx["obs"][t].astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(r[: fx.B].cpu().numpy(), fx["reward"][t].astype(np.float32))
        np.testing.assert_array_equal(d[: fx.B].cpu().numpy(), fx["done"][t].astype(np.uint8))
    st = env.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(st[k][: fx.B], fx[f"final_{k}"], err_msg=k)
    env.check_errors()
    env.close()


def test_device_random_policy_matches_reference():
    from paper_2507_01522_b200.batch import DeviceRandomPolicy

    fx = Fixture("c1_default")
    env = make_env(fx)
    pol = DeviceRandomPolicy(seed=fx.meta["policy_seed"], n_ports=16, k=10)
    pol.bind(range(fx.B))
    for t in range(6):
        np.testing.assert_array_equal(pol.actions(env).cpu().numpy(), fx["actions"][t])
    env.close()


@pytest.mark.parametrize("dtype", ["u8", "i32", "i64", "i64_colmajor"])
def test_action_dtypes_and_strides(dtype):
    fx = Fixture("bp_default")
    env = make_env(fx, obs_dtype=torch.float64)
    env.reset()
    for t in range(20):
        a = torch.as_tensor(fx["actions"][t], device="cuda")
        if dtype == "u8":
            a = a.to(torch.uint8)
        elif dtype == "i32":
            a = a.to(torch.int32)
        elif dtype == "i64_colmajor":
            a = a.t().contiguous().t()
        obs, r, d, _ = env.step(a, collect_infos=False)
        np.testing.assert_array_equal(obs.cpu().numpy(), fx["obs"][t])
    env.close()


def _oracle_subset(tables, B, master, rows, pseed, steps, episode_steps):
    from paper_2507_01522_b200.streams import split_seed

    hb = HostBatch(tables, len(rows), env_seeds=[split_seed(master, i) for i in rows])
    hp = HostRandomPolicy(pseed, tables.n_ports, tables.k, rows)
    frames = [hb.reset()]
    rews = []
    for _ in range(steps):
        o, r, d = hb.step(hp.actions())
        frames.append(o)
        rews.append(r)
    return np.array(frames), np.array(rews), hb


def test_large_batch_subset_matches_oracle():
    """2^16 envs of the default station through an episode boundary; a
    scattered subset of rows is replayed independently on the CPU oracle."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = default_setup()
    B, steps, master, pseed = 1 << 16, 300, 11, 7
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=master)
    pol = DeviceRandomPolicy(pseed, env.n_ports, 10)
    pol.bind(range(B))
    rows = [0, 1, 31, 32, 4095, 4096, 33333, B - 1]
    obs = [env.reset(as_numpy=False)[rows].cpu().numpy()]
    rews = []
    for _ in range(steps):
        o, r, d, _ = env.step(pol.actions(env), collect_infos=False)
        obs.append(o[rows].cpu().numpy())
        rews.append(r[rows].cpu().numpy())
    ref_obs, ref_r, hb = _oracle_subset(env.tables, B, master, rows, pseed, steps, rc.env.episode_steps)
    np.testing.assert_array_equal(np.array(obs), ref_obs.astype(np.float32))
    np.testing.assert_array_equal(np.array(rews), ref_r.astype(np.float32))
    st = env.reference_state()
    for k in ("occ", "soc", "de", "i_drawn", "dtrem", "ep_reward", "ep_profit", "episode", "day"):
        np.testing.assert_array_equal(st[k][rows], getattr(hb.states, k), err_msg=k)
    env.close()


def test_rollout_kernel_equals_stepwise():
    """The fused T-step kernel (state in registers) == T single-step launches."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = default_setup()
    B, T = 3000, 300
    a = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=5)
    b = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=5)
    a.reset(as_numpy=False)
    b.reset(as_numpy=False)
    pol = DeviceRandomPolicy(9, a.n_ports, 10)
    pol.bind(range(B))
    obs_s, rew_s, done_s = [], [], []
    for _ in range(T):
        o, r, d, _ = a.step(pol.actions(a), collect_infos=False)
        obs_s.append(o.clone())
        rew_s.append(r.clone())
        done_s.append(d.clone())
    obs_r = torch.empty(T, B, b.obs_length, device="cuda")
    rew_r = torch.empty(T, B, device="cuda")
    done_r = torch.empty(T, B, dtype=torch.uint8, device="cuda")
    b.rollout(T, 9, 0, obs_r, rew_r, done_r)
    torch.testing.assert_close(obs_r, torch.stack(obs_s), rtol=0, atol=0)
    torch.testing.assert_close(rew_r, torch.stack(rew_s), rtol=0, atol=0)
    torch.testing.assert_close(done_r, torch.stack(done_s), rtol=0, atol=0)
    sa, sb = a.reference_state(), b.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)
    a.close()
    b.close()


@pytest.mark.parametrize("horizon,obs_dtype", [(6, "f32"), (30, "f32"), (4, "f64")])
def test_rollout_generic_horizon_equals_stepwise(horizon, obs_dtype):
    """The generic rollout kernel (price horizon: obs tail of 9 + H columns,
    wider than the per-port chunk ring for H > 3, and beyond one warp for
    H > 23; f64 obs written per lane) equals single steps over an episode
    boundary, ragged last tile included."""
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = default_setup()
    cfg = EnvConfig(observe_price_horizon=horizon)
    dt = torch.float64 if obs_dtype == "f64" else torch.float32
    B, T = 1000, 300
    a = BatchEnv(cfg, rc.station, rc.dataset, batch_size=B, master_seed=2, obs_dtype=dt)
    b = BatchEnv(cfg, rc.station, rc.dataset, batch_size=B, master_seed=2, obs_dtype=dt)
    a.reset(as_numpy=False)
    b.reset(as_numpy=False)
    pol = DeviceRandomPolicy(3, a.n_ports, cfg.discretization_k)
    pol.bind(range(B))
    obs_s, rew_s, done_s = [], [], []
    for _ in range(T):
        o, r, d, _ = a.step(pol.actions(a), collect_infos=False)
        obs_s.append(o.clone())
        rew_s.append(r.clone())
        done_s.append(d.clone())
    obs_r = torch.empty(T, B, b.obs_length, device="cuda", dtype=dt)
    rew_r = torch.empty(T, B, device="cuda", dtype=dt)
    done_r = torch.empty(T, B, dtype=torch.uint8, device="cuda")
    b.rollout(T, 3, 0, obs_r, rew_r, done_r)
    torch.testing.assert_close(obs_r, torch.stack(obs_s), rtol=0, atol=0)
    torch.testing.assert_close(rew_r, torch.stack(rew_s), rtol=0, atol=0)
    torch.testing.assert_close(done_r, torch.stack(done_s), rtol=0, atol=0)
    sa, sb = a.reference_state(), b.reference_state()
    for k in STATE_KEYS:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)
    a.close()
    b.close()


def test_rollout_equals_stepwise_large_tree_lean():
    """Lean instantiations for a large capacity tree (mode 2, nested splitters):
    the fused rollout equals single steps, and a scattered subset of the
    single-step trajectory equals the CPU oracle."""
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy
    from paper_2507_01522_b200.exogenous import generate_synthetic_defaults
    from paper_2507_01522_b200.station import preset_station

    cfg = EnvConfig()
    st = preset_station("nested_splitters", 4, 12)
    ds = generate_synthetic_defaults("highway", "high", "eu", seed=0, days=30)
    B, T, master, pseed = 3072, 300, 4, 6
    a = BatchEnv(cfg, st, ds, batch_size=B, master_seed=master)
    b = BatchEnv(cfg, st, ds, batch_size=B, master_seed=master)
    a.reset(as_numpy=False)
    b.reset(as_numpy=False)
    pol = DeviceRandomPolicy(pseed, a.n_ports, cfg.discretization_k)
    pol.bind(range(B))
    rows = [0, 31, 32, 1000, B - 1]
    obs_s, rew_s = [], []
    for _ in range(T):
        o, r, _, _ = a.step(pol.actions(a), collect_infos=False)
        assert a.last_step_mode() == 2
        obs_s.append(o.clone())
        rew_s.append(r.clone())
    obs_r = torch.empty(T, B, b.obs_length, device="cuda")
    rew_r = torch.empty(T, B, device="cuda")
    done_r = torch.empty(T, B, dtype=torch.uint8, device="cuda")
    b.rollout(T, pseed, 0, obs_r, rew_r, done_r)
    torch.testing.assert_close(obs_r, torch.stack(obs_s), rtol=0, atol=0)
    torch.testing.assert_close(rew_r, torch.stack(rew_s), rtol=0, atol=0)
    ref_obs, ref_r, _ = _oracle_subset(a.tables, B, master, rows, pseed, T, cfg.episode_steps)
    np.testing.assert_array_equal(torch.stack(obs_s)[:, rows].cpu().numpy(), ref_obs[1:].astype(np.float32))
    np.testing.assert_array_equal(torch.stack(rew_s)[:, rows].cpu().numpy(), ref_r.astype(np.float32))
    a.close()
    b.close()


@pytest.mark.parametrize("obs_dtype", ["f32", "f64"])
def test_tree_rescale_every_row_matches_oracle(obs_dtype):
    """Nested splitters (11 nodes, 2-port caps) at high traffic: the tree
    rescale runs multi-pass fixed points on most steps.  Every row and every
    state slot of the kernel (lean mode 2 for f32 obs, the generic kernel for
    f64) equals the CPU oracle over a whole episode and past its boundary."""
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy
    from paper_2507_01522_b200.exogenous import generate_synthetic_defaults
    from paper_2507_01522_b200.station import preset_station

    cfg = EnvConfig()
    st = preset_station("nested_splitters", 4, 12)
    ds = generate_synthetic_defaults("work", "high", "us", seed=2, days=20)
    B, T, master, pseed = 256, 300, 13, 17
    dt = torch.float32 if obs_dtype == "f32" else torch.float64
    env = BatchEnv(cfg, st, ds, batch_size=B, master_seed=master, obs_dtype=dt)
    pol = DeviceRandomPolicy(pseed, env.n_ports, cfg.discretization_k)
    pol.bind(range(B))
    obs = [env.reset(as_numpy=False).cpu().numpy()]
    rews = []
    for _ in range(T):
        o, r, _, _ = env.step(pol.actions(env), collect_infos=False)
        assert env.last_step_mode() == (2 if obs_dtype == "f32" else 0)
        obs.append(o.cpu().numpy())
        rews.append(r.cpu().numpy())
    ref_obs, ref_r, hb = _oracle_subset(env.tables, B, master, list(range(B)), pseed, T, cfg.episode_steps)
    np.testing.assert_array_equal(np.array(obs), ref_obs.astype(obs[0].dtype))
    np.testing.assert_array_equal(np.array(rews), ref_r.astype(rews[0].dtype))
    stt = env.reference_state()
    for k in ("occ", "soc", "de", "i_drawn", "dtrem", "ep_reward", "ep_profit", "episode", "day"):
        np.testing.assert_array_equal(stt[k], getattr(hb.states, k), err_msg=k)
    env.close()


def test_results_invariant_to_launch_shape():
    """The reference's worker-count contract (tests/test_engine.py:78-86) on the
    GPU: the persistent step kernel's grid shape (tiles per warp) does not
    change any output."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    rc = default_setup()
    B = 8192
    envs = [BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=2) for _ in range(3)]
    envs[1].set_tiles_per_warp(3)
    envs[2].set_tiles_per_warp(64)
    pol = DeviceRandomPolicy(5, envs[0].n_ports, 10)
    pol.bind(range(B))
    for e in envs:
        e.reset(as_numpy=False)
    for _ in range(60):
        a = pol.actions(envs[0]).clone()
        outs = [tuple(x.clone() for x in e.step(a, collect_infos=False)[:3]) for e in envs]
        for o in outs[1:]:
            for x, y in zip(outs[0], o):
                torch.testing.assert_close(x, y, rtol=0, atol=0)
    for e in envs:
        e.close()


def test_injected_draws_reproduce_reference_stream():
    """Arrival draws replayed on the host (the reference's own recipe,
    tests/test_env.py:251-278) and injected through vy_draws give the same
    trajectory as the in-kernel reference stream."""
    from paper_2507_01522_b200.exogenous import sample_arrival_count
    from paper_2507_01522_b200.streams import PHASE_ARRIVALS, Stream, stream_key

    fx = Fixture("bp_default")
    ds, sc = fx.dataset, fx.dataset.scenario
    a = make_env(fx, obs_dtype=torch.float64)
    b = make_env(fx, obs_dtype=torch.float64)
    a.reset()
    b.reset()
    for t in range(fx.steps):
        st = b.reference_state()
        draws = {}
        for e in range(fx.B):
            tstep, day = int(st["step"][e]), int(st["day"][e])
            minutes = tstep * fx.config.dt_min
            eff = (day + minutes // 1440) % ds.prices.n_days
            scale = ds.arrivals.weekday_scale if ds.prices.is_weekday(eff) else ds.arrivals.weekend_scale
            lam = float(ds.arrivals.rates_per_step[tstep % len(ds.arrivals.rates_per_step)]) * scale
            s = Stream(stream_key(int(st["env_seed"][e]), int(st["episode"][e]), PHASE_ARRIVALS, tstep))
            rows = []
            for _ in range(sample_arrival_count(s, lam)):
                kcar = s.choice_cum(ds.cars.cumulative_weights())
                lo, hi = sc.stay_steps_range
                stay = lo + s.randint(hi - lo + 1)
                soc0 = sc.soc_arrival_range[0] + s.uniform() * (sc.soc_arrival_range[1] - sc.soc_arrival_range[0])
                frac = sc.requested_fraction_range[0] + s.uniform() * (
                    sc.requested_fraction_range[1] - sc.requested_fraction_range[0])
                rows.append((kcar, stay, soc0, frac, s.bernoulli(sc.p_charge_sensitive)))
            draws[e] = rows
        oa, ra, da, _ = a.step(fx["actions"][t], collect_infos=False)
        ob, rb, db = b.step_injected(fx["actions"][t], draws)
        np.testing.assert_array_equal(ob.cpu().numpy(), oa, err_msg=f"t={t}")
        np.testing.assert_array_equal(rb.cpu().numpy(), ra)
    a.close()
    b.close()


def test_errors_match_reference_behaviour():
    from paper_2507_01522_b200.errors import EpisodeDone

    fx = Fixture("bp_default")
    env = make_env(fx)
    with pytest.raises(EpisodeDone):
        env.step(fx["actions"][0])
    env.reset()
    with pytest.raises(ValueError):
        env.step(np.zeros((fx.B + 1, fx.station.n_ports + 1), dtype=np.int64))
    bad = fx["actions"][0].copy()
    bad[0, 0] = 21
    with pytest.raises(ValueError):
        env.step(bad)
    # device path: detected on the GPU, raised at the next synchronising call
    env.step(torch.as_tensor(bad, device="cuda"), collect_infos=False)
    with pytest.raises(ValueError):
        env.check_errors()
    env.check_errors()  # cleared
    env.close()


def test_host_path_returns_fresh_arrays_and_accepts_any_int_actions():
    """The numpy drop-in returns new float64/bool arrays every step (callers
    keep them, as the reference's .copy() allows, engine.py:463-464) and takes
    read-only or narrower integer action arrays like np.ascontiguousarray."""
    fx = Fixture("bp_default")
    env = make_env(fx, obs_dtype=torch.float64)
    obs0 = env.reset()
    a0 = fx["actions"][0].astype(np.int32)
    a0.setflags(write=False)
    obs1, r1, d1, _ = env.step(a0, collect_infos=False)
    keep = obs1.copy(), r1.copy(), d1.copy()
    obs2, r2, d2, _ = env.step(fx["actions"][1], collect_infos=False)
    assert obs1.dtype == np.float64 and r1.dtype == np.float64 and d1.dtype == np.bool_
    assert not np.shares_memory(obs1, obs2) and not np.shares_memory(obs0, obs1)
    np.testing.assert_array_equal(obs1, keep[0])
    np.testing.assert_array_equal(r1, keep[1])
    np.testing.assert_array_equal(d1, keep[2])
    np.testing.assert_array_equal(obs0, fx["obs0"])
    np.testing.assert_array_equal(obs1, fx["obs"][0])
    np.testing.assert_array_equal(obs2, fx["obs"][1])
    neg = fx["actions"][2].copy()
    neg[-1, -1] = -1
    with pytest.raises(ValueError):
        env.step(neg)
    env.close()


def test_no_auto_reset_raises_episode_done():
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.errors import EpisodeDone

    fx = Fixture("bp_default")
    from paper_2507_01522_b200 import EnvConfig

    cfg = EnvConfig(episode_steps=5)
    env = BatchEnv(cfg, fx.station, fx.dataset, batch_size=2, auto_reset=False)
    env.reset()
    idle = np.full((2, fx.station.n_ports + 1), 10, dtype=np.int64)
    for _ in range(5):
        _, _, d, _ = env.step(idle, collect_infos=False)
    assert d.all()
    with pytest.raises(EpisodeDone):
        env.step(idle)
    env.close()


def test_injected_car_known_answers():
    """Clipping / flow known answers of the reference (tests/test_env.py:48-128)."""
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import BatchEnv
    from scenarios import single_node_station, make_dataset

    # target 15 vs rate-equivalent 375 A vs port max 16 A -> 15
    env = BatchEnv(EnvConfig(discretization_k=16), single_node_station(n_ports=1, i_max=16.0, voltage_v=400.0),
                   make_dataset(), batch_size=1, auto_reset=False, obs_dtype=torch.float64)
    env.reset()
    env.inject_car(0, soc=0.5, r_bar=150.0, i_drawn=10.0)
    a = np.full((1, 2), 16, dtype=np.int64)
    a[0, 0] = 21
    _, _, _, infos = env.step(a)
    assert infos[0].currents_applied_a[0] == pytest.approx(15.0, rel=1e-12)
    env.close()
    # flows: 5/3 kWh delivered at 20 A * 1000 V over 5 min, eta_c 0.9 -> e_in = (5/3)/0.9
    env = BatchEnv(EnvConfig(), single_node_station(n_ports=1, voltage_v=1000.0, i_max=20.0, eta_charge=0.9),
                   make_dataset(), batch_size=1, auto_reset=False, obs_dtype=torch.float64)
    env.reset()
    env.inject_car(0, soc=0.1, cap=100.0, r_bar=150.0, de=100.0, i_drawn=20.0)
    _, _, _, infos = env.step(np.array([[10, 10]]))
    assert infos[0].flows.e_net == pytest.approx(5.0 / 3.0, rel=1e-12)
    assert infos[0].flows.e_grid_in == pytest.approx((5.0 / 3.0) / 0.9, rel=1e-12)
    env.close()


def test_numpy_outputs_are_owned_by_the_caller():
    """The exact numpy path hands out pinned ring buffers: arrays a caller
    keeps are never overwritten by later steps (reference semantics: fresh
    copies, engine.py:463-464), and the steady state reuses the ring."""
    fx = Fixture("c1_default")
    env = make_env(fx, obs_dtype=torch.float64)
    env.reset()
    kept = []
    for t in range(12):
        obs, r, d, _ = env.step(fx["actions"][t], collect_infos=False)
        kept.append((t, obs, r, d))
    for t, obs, r, d in kept:
        np.testing.assert_array_equal(obs, fx["obs"][t], err_msg=f"kept obs t={t}")
        np.testing.assert_array_equal(r, fx["reward"][t])
        np.testing.assert_array_equal(d.astype(np.int8), fx["done"][t])
    kept.clear()
    ids = set()
    for t in range(12, 30):
        obs, r, d, _ = env.step(fx["actions"][t], collect_infos=False)
        np.testing.assert_array_equal(obs, fx["obs"][t], err_msg=f"t={t}")
        ids.add(obs.ctypes.data)
    assert len(ids) <= 4  # ring buffers, not a fresh allocation per step
    env.close()
