"""Rebuild golden-fixture scenarios with this package's own host types.

Fixtures (tests/golden/*.npz, made by scripts/make_golden.py from the
reference) carry their inputs, so nothing here needs /root/reference.
"""

from __future__ import annotations

import datetime as dt
import json
from pathlib import Path

import numpy as np

from paper_2507_01522_b200.envconfig import EnvConfig
from paper_2507_01522_b200.exogenous import (ArrivalProfile, AuxSeries, CarCatalog, CatalogEntry, Dataset,
                                             PriceSeries, UserScenarioModel)
from paper_2507_01522_b200.physics import CarProfile
from paper_2507_01522_b200.station import station_from_dict
from paper_2507_01522_b200.tables import build_tables

GOLDEN = Path(__file__).resolve().parent / "golden"
NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem not in ("synthetic_vectors", "bridge_spaces"))


class Fixture:
    def __init__(self, name: str):
        z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
        self.z = z
        self.meta = json.loads(str(z["meta"]))
        self.name = name
        self.config = EnvConfig.from_dict(self.meta["config"])
        self.station = station_from_dict(self.meta["station"])
        sc = z["ds_scenario"]
        aux = AuxSeries(z["ds_moer"] if "ds_moer" in z else None, z["ds_dgrid"] if "ds_dgrid" in z else None)
        cars = CarCatalog(tuple(CatalogEntry(CarProfile(*row[:4]), float(row[4])) for row in z["ds_cars"]))
        self.dataset = Dataset(
            prices=PriceSeries(dt.date.fromisoformat(str(z["ds_start_date"])), z["ds_buy"], z["ds_sell_grid"]),
            arrivals=ArrivalProfile(z["ds_rates"], float(z["ds_scales"][0]), float(z["ds_scales"][1])),
            cars=cars,
            scenario=UserScenarioModel((int(sc[0]), int(sc[1])), (sc[2], sc[3]), (sc[4], sc[5]), float(sc[6])),
            aux=aux,
        )
        self.B = self.meta["batch"]
        self.master_seed = self.meta["master_seed"]
        self.steps = self.meta["steps"]

    def tables(self):
        return build_tables(self.config, self.station, self.dataset)

    def __getitem__(self, k):
        return self.z[k]


# --- small builders (same parameters as the reference's tests/helpers.py:22-101) ---

def make_dataset(lam: float = 0.0, buy: float = 0.10, sell_grid=None, days: int = 3, dt_min: int = 5,
                 stay_range=(6, 24), frac_range=(0.3, 0.9), soc_range=(0.2, 0.7), p_charge: float = 0.3,
                 cars=None, moer=None, grid_demand=None) -> Dataset:
    n = days * 24
    cars = cars or CarCatalog((CatalogEntry(CarProfile(60.0, 11.0, 120.0, 0.8, name="a"), 1.0),
                               CatalogEntry(CarProfile(40.0, 7.4, 60.0, 0.8, name="b"), 1.0)))
    return Dataset(
        prices=PriceSeries(dt.date(2022, 1, 3), np.full(n, buy), np.full(n, buy if sell_grid is None else sell_grid)),
        arrivals=ArrivalProfile(np.full(1440 // dt_min, lam)),
        cars=cars,
        scenario=UserScenarioModel(stay_range, frac_range, soc_range, p_charge),
        aux=AuxSeries(None if moer is None else np.full(n, moer),
                      None if grid_demand is None else np.full(n, grid_demand)),
    )


def single_node_station(n_ports: int = 2, cap_a: float = 1e9, voltage_v: float = 400.0, i_max: float = 400.0,
                        i_max_discharge=None, eta_charge: float = 1.0, eta_discharge: float = 1.0,
                        kind: str = "dc", node_eta: float = 1.0, battery=None):
    from paper_2507_01522_b200.station import ArchNode, EvseSpec, build_station

    leaves = tuple(EvseSpec(id=i, voltage_v=voltage_v, i_max_charge_a=i_max,
                            i_max_discharge_a=i_max if i_max_discharge is None else i_max_discharge,
                            eta_charge=eta_charge, eta_discharge=eta_discharge, kind=kind) for i in range(n_ports))
    return build_station(ArchNode(capacity_a=cap_a, eta=node_eta, children=leaves), battery=battery)


def random_station(rng: np.random.Generator, max_depth: int = 3, max_leaves: int = 8, battery=None, types=None):
    """A random capacity tree with binding capacities — the generator of the
    reference's constraint suite (tests/helpers.py:104-160) restated: up to
    ``max_leaves`` ports (AC or DC, 230-800 V, 16-400 A, 30% charge-only,
    eta 0.85-1), internal nodes of 2-3 children at capacity 0.2-1.2x their
    subtree's charge current, half of them lossy (eta 0.8-1).  ``types``: a
    namespace with ArchNode / EvseSpec / build_station (default: this
    package's; ref_scenarios passes the reference's)."""
    if types is None:
        from paper_2507_01522_b200 import station as types
    ArchNode, EvseSpec, build_station = types.ArchNode, types.EvseSpec, types.build_station

    ids = iter(range(1 << 20))
    budget = [int(rng.integers(1, max_leaves + 1))]

    def port():
        budget[0] -= 1
        dc = rng.random() < 0.5
        imax = float(rng.uniform(16, 400))
        return EvseSpec(id=next(ids), voltage_v=float(rng.uniform(230, 800)), i_max_charge_a=imax,
                        i_max_discharge_a=imax if rng.random() < 0.7 else 0.0,
                        eta_charge=float(rng.uniform(0.85, 1.0)), eta_discharge=float(rng.uniform(0.85, 1.0)),
                        kind="dc" if dc else "ac")

    def amps(nodes):
        return sum(n.i_max_charge_a if isinstance(n, EvseSpec) else amps(n.children) for n in nodes)

    def subtree(depth):
        if depth >= max_depth or budget[0] <= 1 or rng.random() < 0.3:
            return port()
        kids = []
        for _ in range(int(rng.integers(2, 4))):
            if budget[0] <= 0:
                break
            kids.append(subtree(depth + 1))
        if not kids:
            return port()
        eta = float(rng.uniform(0.8, 1.0)) if rng.random() < 0.5 else 1.0
        return ArchNode(capacity_a=float(rng.uniform(0.2, 1.2) * max(amps(kids), 1.0)), eta=eta,
                        children=tuple(kids))

    top = [subtree(1)]
    while budget[0] > 0:
        top.append(subtree(1))
    root = ArchNode(capacity_a=float(rng.uniform(0.2, 1.2) * max(amps(top), 1.0)), eta=1.0, children=tuple(top))
    return build_station(root, battery=battery)
