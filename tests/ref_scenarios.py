"""The six scenarios of the reference's backend-parity test
(pkg/tests/test_backend_parity.py:23-34) built from the reference's own types
(the installed package in baseline/_ref), for the plugin tests that drive the
reference's unmodified BatchEnv.  The builders restate pkg/tests/helpers.py:22-101
(make_dataset, single_node_station) over those types; the random tree comes
from scenarios.random_station with the reference's classes."""

from __future__ import annotations

import datetime as dt
import sys
from pathlib import Path

import numpy as np

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def import_reference():
    """The installed reference package, or None when baseline/_ref is absent."""
    if not (REF / "voltyard").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import voltyard

    return voltyard


def make_dataset(lam=0.0, buy=0.10, days=3, dt_min=5, moer=None, grid_demand=None):
    from voltyard.data import ArrivalProfile, AuxSeries, CarCatalog, CatalogEntry, Dataset, PriceSeries, \
        UserScenarioModel
    from voltyard.vehicles import CarProfile

    n = days * 24
    return Dataset(
        prices=PriceSeries(start_date=dt.date(2022, 1, 3), buy=np.full(n, buy), sell_grid=np.full(n, buy),
                           region="flat"),
        arrivals=ArrivalProfile(rates_per_step=np.full(1440 // dt_min, lam), scenario="test"),
        cars=CarCatalog(entries=(CatalogEntry(CarProfile(60.0, 11.0, 120.0, 0.8, name="a"), 1.0),
                                 CatalogEntry(CarProfile(40.0, 7.4, 60.0, 0.8, name="b"), 1.0)), region="test"),
        scenario=UserScenarioModel(stay_steps_range=(6, 24), requested_fraction_range=(0.3, 0.9),
                                   soc_arrival_range=(0.2, 0.7), p_charge_sensitive=0.3, scenario="test"),
        aux=AuxSeries(moer_kg_per_kwh=np.full(n, moer) if moer is not None else None,
                      grid_demand_kwh=np.full(n, grid_demand) if grid_demand is not None else None),
    )


def single_node_station(n_ports=2, cap_a=1e9, voltage_v=400.0, i_max=400.0, eta_charge=1.0, eta_discharge=1.0,
                        battery=None):
    from voltyard.topology import ArchNode, EvseSpec, build_station

    leaves = tuple(EvseSpec(id=i, voltage_v=voltage_v, i_max_charge_a=i_max, i_max_discharge_a=i_max,
                            eta_charge=eta_charge, eta_discharge=eta_discharge, kind="dc") for i in range(n_ports))
    return build_station(ArchNode(capacity_a=cap_a, eta=1.0, children=leaves), battery=battery)


def scenario_cases():
    """test_backend_parity.py:23-34, same parameters."""
    from voltyard import topology
    from voltyard.config import EnvConfig
    from voltyard.topology import preset_station
    from voltyard.vehicles import BatterySpec

    from scenarios import random_station

    batt = BatterySpec(voltage_v=800.0, capacity_kwh=120.0, r_max_kw=60.0, tau=0.75, eta_charge=0.95,
                       eta_discharge=0.93)
    yield "default", EnvConfig(episode_steps=96), single_node_station(n_ports=4, cap_a=600.0), make_dataset(lam=2.0)
    yield "battery+penalties", EnvConfig(
        episode_steps=96, battery_enabled=True, battery_init_soc=0.4, beta=0.5,
        alpha={"constraint": 0.1, "sat0": 0.2, "sat1": 0.3, "sustain": 0.4, "declined": 0.5,
               "degrad_battery": 0.6, "degrad_cars": 0.7, "grid": 0.8}), \
        single_node_station(n_ports=3, cap_a=300.0, eta_charge=0.92, eta_discharge=0.9, battery=batt), \
        make_dataset(lam=2.5, moer=0.35, grid_demand=3.0)
    yield "no-discharge", EnvConfig(episode_steps=64, allow_discharge=False), \
        single_node_station(n_ports=3, cap_a=200.0), make_dataset(lam=1.0)
    yield "nested-station", EnvConfig(episode_steps=64, discretization_k=4, observe_price_horizon=6), \
        preset_station("nested_splitters", 4, 4), make_dataset(lam=3.0)
    yield "coarse-dt", EnvConfig(episode_steps=96, dt_min=15), single_node_station(n_ports=2), \
        make_dataset(lam=1.0, dt_min=15)
    yield "random-tree", EnvConfig(episode_steps=64), \
        random_station(np.random.default_rng(99), types=topology), make_dataset(lam=2.0)
