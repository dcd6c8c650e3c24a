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
NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "synthetic_vectors")


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
