"""Generate golden fixtures from the reference implementation itself.

Runs ONLY in the build container (needs /root/reference).  Imports voltyard
from a scratch build of /root/reference/pkg (compiled Cython kernel when
available, else the bit-identical pure-Python kernel), runs the scenarios
below through the reference's own BatchEnv + RandomPolicy/MaxChargePolicy,
and writes tests/golden/<name>.npz holding

  * the scenario inputs (config dict, station dict, dataset arrays, seeds),
  * the reference's build_tables() output (pins our tables.py),
  * the actions fed, and every per-step output the engine exposes.

The GPU box has no /root/reference: tests rebuild each scenario from the
fixture alone.  Usage:  python scripts/make_golden.py [--ref /tmp/vyref/src]
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"


def ensure_ref(path: str | None) -> str:
    if path:
        return path
    scratch = Path("/tmp/vyref")
    if not (scratch / "src" / "voltyard").exists():
        shutil.copytree("/root/reference/pkg", scratch)
        subprocess.run(["chmod", "-R", "u+w", str(scratch)], check=True)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=scratch, check=True,
                       stdout=subprocess.DEVNULL)
    return str(scratch / "src")


def scenarios(vy, helpers):
    EnvConfig, BatterySpec = vy.EnvConfig, vy.BatterySpec
    mk, single, rnd = helpers.make_dataset, helpers.single_node_station, helpers.random_station
    batt = BatterySpec(voltage_v=800.0, capacity_kwh=120.0, r_max_kw=60.0, tau=0.75,
                       eta_charge=0.95, eta_discharge=0.93)
    all_alpha = {"constraint": 0.1, "sat0": 0.2, "sat1": 0.3, "sustain": 0.4,
                 "declined": 0.5, "degrad_battery": 0.6, "degrad_cars": 0.7, "grid": 0.8}
    # the six backend-parity scenarios (tests/test_backend_parity.py:23-34)
    yield "bp_default", EnvConfig(episode_steps=96), single(n_ports=4, cap_a=600.0), mk(lam=2.0), 3, 17, 23, "random", 192
    yield "bp_battery_penalties", EnvConfig(episode_steps=96, battery_enabled=True, battery_init_soc=0.4, beta=0.5,
                                            alpha=all_alpha), \
        single(n_ports=3, cap_a=300.0, eta_charge=0.92, eta_discharge=0.9, battery=batt), \
        mk(lam=2.5, moer=0.35, grid_demand=3.0), 3, 17, 23, "random", 192
    yield "bp_no_discharge", EnvConfig(episode_steps=64, allow_discharge=False), single(n_ports=3, cap_a=200.0), \
        mk(lam=1.0), 3, 17, 23, "random", 128
    yield "bp_nested", EnvConfig(episode_steps=64, discretization_k=4, observe_price_horizon=6), \
        vy.preset_station("nested_splitters", 4, 4), mk(lam=3.0), 3, 17, 23, "random", 128
    yield "bp_coarse_dt", EnvConfig(episode_steps=96, dt_min=15), single(n_ports=2), mk(lam=1.0, dt_min=15), \
        3, 17, 23, "random", 192
    yield "bp_random_tree", EnvConfig(episode_steps=64), rnd(np.random.default_rng(99)), mk(lam=2.0), \
        3, 17, 23, "random", 128
    # config C1 literally: default station, 16 envs x 288 steps (+ crossing the auto-reset)
    rc = vy.default_setup()
    yield "c1_default", rc.env, rc.station, rc.dataset, 16, 0, 0, "random", 300
    # saturating policy: exercises the tree rescale every step
    yield "default_maxcharge", rc.env, rc.station, rc.dataset, 4, 5, 0, "max_charge", 200
    # config C4 shape: 64 DC ports, 3-level splitter tree, battery, profit + satisfaction reward
    cfg4 = EnvConfig(battery_enabled=True, alpha={"sat0": 1.0, "sat1": 0.5}, beta=0.2)
    st4 = vy.preset_station("nested_splitters", ac_count=0, dc_count=64, battery=vy.DEFAULT_BATTERY)
    ds4 = vy.generate_synthetic_defaults("highway", "high", "eu", seed=0)
    yield "c4_highway64", cfg4, st4, ds4, 2, 3, 1, "random", 120
    # aux series (MOER + grid demand), all penalties, fixed cost, world region catalogue
    cfg_aux = EnvConfig(episode_steps=96, alpha=all_alpha, beta=0.3, fixed_cost_per_step=0.05)
    rca = vy.default_setup(cfg_aux, scenario="work", traffic="high", region="world", seed=4, days=30, with_aux=True)
    yield "aux_all_penalties", rca.env, rca.station, rca.dataset, 3, 9, 2, "random", 150
    # non-identity parking order + AC-only single node
    leaves = tuple(vy.EvseSpec(id=i, voltage_v=230.0, i_max_charge_a=32.0, i_max_discharge_a=16.0,
                               eta_charge=0.9, eta_discharge=0.85) for i in range(5))
    st_po = vy.build_station(vy.ArchNode(capacity_a=70.0, children=leaves), evse_order=[3, 1, 4, 0, 2])
    yield "parking_order", EnvConfig(episode_steps=48), st_po, mk(lam=1.5, days=4), 3, 21, 4, "random", 96
    # whole 32-env tiles, so the GPU tests run these through the lean step
    # instantiations as well: C5-style stations and markets (config C5 groups)
    # and the C2 station, each crossing an episode boundary
    cfg96 = EnvConfig(episode_steps=96)
    yield "c5_nested_residential_us", cfg96, vy.preset_station("nested_splitters", 4, 12), \
        vy.generate_synthetic_defaults("residential", "low", "us", seed=0, days=20), 32, 6, 8, "random", 150
    yield "c5_single_highway_world", cfg96, vy.preset_station("single_type", 0, 8), \
        vy.generate_synthetic_defaults("highway", "high", "world", seed=0, days=20), 32, 7, 9, "random", 150
    yield "c2_default_tile", cfg96, rc.station, vy.generate_synthetic_defaults("shopping", "medium", "eu", seed=0,
                                                                                 days=20), 32, 8, 10, "random", 150


def dataset_dict(ds) -> dict:
    d = {
        "start_date": ds.prices.start_date.isoformat(),
        "buy": ds.prices.buy, "sell_grid": ds.prices.sell_grid,
        "rates": ds.arrivals.rates_per_step,
        "scales": np.array([ds.arrivals.weekday_scale, ds.arrivals.weekend_scale]),
        "cars": np.array([[e.profile.capacity_kwh, e.profile.r_max_ac_kw, e.profile.r_max_dc_kw,
                           e.profile.tau, e.weight] for e in ds.cars.entries]),
        "scenario": np.array([*ds.scenario.stay_steps_range, *ds.scenario.requested_fraction_range,
                              *ds.scenario.soc_arrival_range, ds.scenario.p_charge_sensitive]),
    }
    if ds.aux.moer_kg_per_kwh is not None:
        d["moer"] = ds.aux.moer_kg_per_kwh
    if ds.aux.grid_demand_kwh is not None:
        d["dgrid"] = ds.aux.grid_demand_kwh
    return d


def run(vy, name, cfg, station, ds, B, master, pseed, policy, steps):
    from voltyard.engine import build_tables

    env = vy.BatchEnv(cfg, station, ds, batch_size=B, master_seed=master)
    pol = vy.make_policy(policy, station.n_ports, cfg.discretization_k, seed=pseed)
    pol.bind(range(B))
    obs = env.reset()
    rec: dict[str, list] = {k: [] for k in (
        "actions", "obs", "reward", "done", "breakdown", "flows", "declined", "arrivals_m", "dep_n",
        "dep_port", "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc",
        "term_overtime", "i_att", "i_used", "delivered", "b_delivered", "ep_stats", "step", "day", "episode")}
    obs0 = obs.copy()
    o, s = env.outs, env.states
    for _ in range(steps):
        a = pol.actions(obs)
        obs, r, d, _ = env.step(a, collect_infos=False)
        rec["actions"].append(a.astype(np.int64))
        rec["obs"].append(obs.copy())
        rec["reward"].append(r.copy())
        rec["done"].append(d.astype(np.int8))
        for k in ("breakdown", "flows", "declined", "arrivals_m", "dep_n", "dep_port", "dep_missing",
                  "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc", "term_overtime",
                  "i_att", "i_used", "delivered", "b_delivered"):
            rec[k].append(getattr(o, k).copy())
        rec["ep_stats"].append(np.where(d[:, None], o.ep_stats, 0.0))
        rec["step"].append(s.step.copy())
        rec["day"].append(s.day.copy())
        rec["episode"].append(s.episode.copy())
    # dep_* rows beyond dep_n are stale by design; mask them so fixtures hold only defined entries
    dn = np.array(rec["dep_n"])
    for k in ("dep_port", "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc"):
        arr = np.array(rec[k])
        mask = np.arange(arr.shape[-1])[None, None, :] < dn[:, :, None]
        rec[k] = np.where(mask, arr, 0)
    final = {f"final_{k}": getattr(s, k).copy() for k in (
        "occ", "i_drawn", "soc", "de", "dtrem", "cap", "rbar", "tau", "pref", "rhat", "b_i", "b_soc", "b_rhat",
        "step", "day", "episode", "env_seed", "ep_profit", "ep_reward", "ep_missing", "ep_energy",
        "ep_overtime", "ep_declined", "ep_departures")}
    env.close()
    tabs = build_tables(cfg, station, ds)
    tab = {}
    for k, v in vars(tabs).items():
        tab[f"tab_{k}"] = np.asarray(v)
    meta = {
        "name": name, "config": cfg.to_dict(), "station": vy.topology.station_to_dict(station),
        "batch": B, "master_seed": master, "policy": policy, "policy_seed": pseed, "steps": steps,
        "backend": env.backend,
    }
    payload = {"meta": np.array(json.dumps(meta)), "obs0": obs0}
    payload.update({f"ds_{k}": np.asarray(v) for k, v in dataset_dict(ds).items()})
    payload.update({k: np.array(v) for k, v in rec.items()})
    payload.update(final)
    payload.update(tab)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **payload)
    return env.backend


def synthetic_vectors(vy):
    """Synthetic generators' arrays for several (scenario, traffic, region, seed)."""
    out = {}
    for sc in ("highway", "residential", "work", "shopping"):
        for tr in ("low", "medium", "high"):
            a = vy.data.synthetic_arrivals(sc, tr, dt_min=5)
            out[f"arr_{sc}_{tr}"] = a.rates_per_step
            out[f"arrscale_{sc}_{tr}"] = np.array([a.weekday_scale, a.weekend_scale])
        for dtm in (1, 5, 15):
            m = vy.data.scenario_model(sc, dt_min=dtm)
            out[f"scen_{sc}_{dtm}"] = np.array([*m.stay_steps_range, *m.requested_fraction_range,
                                                *m.soc_arrival_range, m.p_charge_sensitive])
    for rg in ("eu", "us", "world"):
        for seed in (0, 7):
            p = vy.data.synthetic_prices(rg, seed=seed, days=40)
            out[f"price_{rg}_{seed}"] = p.buy
            out[f"sell_{rg}_{seed}"] = p.sell_grid
        c = vy.data.car_catalog(rg)
        out[f"cum_{rg}"] = c.cumulative_weights()
    aux = vy.data.synthetic_aux(seed=3, days=20)
    out["aux_moer_3"], out["aux_dgrid_3"] = aux.moer_kg_per_kwh, aux.grid_demand_kwh
    # RNG known answers
    from voltyard import rng
    keys = [rng.stream_key(11, i) for i in range(64)]
    out["rng_keys"] = np.array(keys, dtype=np.uint64)
    st = rng.BatchStreams(np.array(keys, dtype=np.uint64))
    out["rng_u"] = st.uniform_block(9)
    out["rng_pois"] = np.array([rng.Stream(k).poisson(3.7) for k in keys])
    out["rng_pois_big"] = np.array([rng.Stream(k).poisson(70.5) for k in keys])
    out["split_seed"] = np.array([rng.split_seed(m, i) for m in (-17, 0, 42) for i in range(8)], dtype=np.uint64)
    pol = vy.RandomPolicy(seed=5, n_ports=16, k=10)
    pol.bind(range(1000, 1032))
    out["policy_actions"] = np.stack([pol.actions(np.zeros((32, 105))) for _ in range(3)])
    np.savez_compressed(OUT / "synthetic_vectors.npz", **out)


def evaluate_vectors(vy):
    """evaluate() reports of the three baseline policies (evaluate.py:78-142)."""
    from voltyard.evaluate import evaluate

    rc = vy.default_setup(vy.EnvConfig(episode_steps=96), days=40)
    out = {}
    for name in ("max_charge", "idle", "random"):
        rep = evaluate(vy.make_policy(name, 16, 10, seed=3), rc.env, rc.station, rc.dataset, episodes=150, seed=7)
        out[name] = rep.to_dict()
    cfg4 = vy.EnvConfig(episode_steps=48, battery_enabled=True, alpha={"sat0": 1.0}, beta=0.1)
    rc4 = vy.default_setup(cfg4, scenario="highway", traffic="high", days=20)
    out["max_charge_battery"] = evaluate(vy.make_policy("max_charge", 16, 10), rc4.env, rc4.station, rc4.dataset,
                                         episodes=40, seed=2).to_dict()
    (OUT / "evaluate_reports.json").write_text(json.dumps(out, indent=1, sort_keys=True))


def bridge_vectors(vy):
    """Observation-space bounds of the reference bridge (voltyard_gym :74-97)."""
    sys.path.insert(0, "/root/reference/pkg/bridge/src")
    from voltyard_gym import ChargingVectorEnv

    out = {}
    for tag, cfg, station, kw in (
            ("default", vy.EnvConfig(), None, {}),
            ("c4", vy.EnvConfig(battery_enabled=True), vy.preset_station("nested_splitters", ac_count=0, dc_count=64,
                                                                         battery=vy.DEFAULT_BATTERY), {})):
        rc = vy.default_setup(cfg, days=10, **kw)
        env = ChargingVectorEnv(rc.env, station or rc.station, rc.dataset, num_envs=1, seed=0)
        out[f"{tag}_low"] = env.observation_space.low
        out[f"{tag}_high"] = env.observation_space.high
        env.close()
    np.savez_compressed(OUT / "bridge_spaces.npz", **out)


BAD_FILES = {
    # name: (file, contents, loader)
    "prices_gap": ("prices.csv", "timestamp,buy_eur_per_kwh\n2023-01-01T00:00,0.1\n2023-01-01T02:00,0.2\n", "load_prices"),
    "prices_dup": ("prices.csv", "timestamp,buy_eur_per_kwh\n2023-01-01T00:00,0.1\n2023-01-01T00:00,0.2\n", "load_prices"),
    "prices_offhour": ("prices.csv", "timestamp,buy_eur_per_kwh\n2023-01-01T00:30,0.1\n", "load_prices"),
    "prices_col": ("prices.csv", "time,buy\n2023-01-01T00:00,0.1\n", "load_prices"),
    "prices_empty": ("prices.csv", "timestamp,buy_eur_per_kwh\n", "load_prices"),
    "prices_parse": ("prices.csv", "timestamp,buy_eur_per_kwh\n2023-01-01T00:00,abc\n", "load_prices"),
    "arrivals_order": ("arrivals.csv", "step_of_day,lambda\n0,0.1\n2,0.2\n", "load_arrivals"),
    "arrivals_neg": ("arrivals.csv", "step_of_day,lambda\n0,-0.1\n", "load_arrivals"),
    "cars_tau": ("cars.csv", "name,capacity_kwh,r_max_ac_kw,r_max_dc_kw,tau,weight\nx,50,11,100,1.5,1\n",
                 "load_car_catalog"),
    "cars_cap": ("cars.csv", "name,capacity_kwh,r_max_ac_kw,r_max_dc_kw,tau,weight\nx,0,11,100,0.8,1\n",
                 "load_car_catalog"),
    "cars_zero": ("cars.csv", "name,capacity_kwh,r_max_ac_kw,r_max_dc_kw,tau,weight\nx,50,11,100,0.8,0\n",
                  "load_car_catalog"),
    "aux_cols": ("aux.csv", "timestamp,foo\n2023-01-01T00:00,1\n", "load_aux"),
}


def ingest_vectors(vy):
    """Dataset directory + station JSON written by the reference, and its loader errors."""
    import tempfile

    from voltyard import data as vd
    from voltyard import topology as vt

    d = OUT / "ingest"
    d.mkdir(exist_ok=True)
    import dataclasses

    ds = vy.generate_synthetic_defaults("work", "high", "us", seed=5, days=3)
    ds = dataclasses.replace(ds, aux=vd.synthetic_aux(seed=1, days=3))
    vd.save_dataset(ds, d / "dataset")
    st = vy.preset_station("nested_splitters", ac_count=4, dc_count=6, battery=vy.DEFAULT_BATTERY)
    obj = vt.station_to_dict(st)
    obj["evse_order"] = list(reversed([e.id for e in st.evses]))
    vt.save_station(vt.station_from_dict(obj), d / "station.json")
    errs = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (fname, text, loader) in BAD_FILES.items():
            p = Path(tmp) / fname
            p.write_text(text)
            case = {"file": fname, "text": text, "loader": loader, "error": None}
            try:
                getattr(vd, loader)(p)
            except vy.DataError as exc:
                case["error"] = str(exc).replace(str(p), "<path>")
            errs[name] = case
    (d / "errors.json").write_text(json.dumps(errs, indent=1, sort_keys=True))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=None)
    ap.add_argument("--only", nargs="*", default=None, help="regenerate only these scenarios (no vectors)")
    args = ap.parse_args()
    sys.path.insert(0, ensure_ref(args.ref))
    sys.path.insert(0, "/root/reference/pkg/tests")
    import voltyard as vy  # noqa: E402
    import voltyard.data  # noqa: F401,E402
    import voltyard.topology  # noqa: F401,E402
    import helpers  # noqa: E402

    print("reference backends:", vy.available_backends())
    for sc in scenarios(vy, helpers):
        if args.only is not None and sc[0] not in args.only:
            continue
        be = run(vy, *sc)
        print("wrote", sc[0], "backend", be)
    if args.only is not None:
        return
    synthetic_vectors(vy)
    print("wrote synthetic_vectors")
    evaluate_vectors(vy)
    bridge_vectors(vy)
    ingest_vectors(vy)
    print("wrote evaluate_reports")


if __name__ == "__main__":
    main()
