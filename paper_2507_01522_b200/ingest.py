"""Host data ingestion: dataset CSV directories and station JSON.

File formats and validation rules follow the reference loaders
(``voltyard/data.py:266-527``, ``voltyard/topology.py:498-506``) so a dataset
directory or station file written by either side loads on the other and
produces identical step tables:

* ``prices.csv``   — ``timestamp, buy_eur_per_kwh[, sell_grid_eur_per_kwh]``,
  hourly, starting on the hour, no gaps / duplicates (``data.py:280-315``);
* ``arrivals.csv`` — ``step_of_day, lambda``, steps 0,1,2,…, rates ≥ 0
  (``:328-351``);
* ``cars.csv``     — ``name, capacity_kwh, r_max_ac_kw, r_max_dc_kw, tau,
  weight`` (``:362-397``);
* ``aux.csv``      — ``timestamp`` + ``moer_kg_per_kwh`` and/or
  ``grid_demand_kwh`` (``:412-436``), optional;
* ``scenario.json`` — user-scenario model + arrival-day multipliers
  (``:465-499``), optional (shopping defaults).

Writers emit ``repr`` floats so a save → load round trip is exact.  Errors
are ``DataError`` with ``path: message at line N``, as in the reference.
"""

from __future__ import annotations

import csv
import datetime as dt
import json
from pathlib import Path

import numpy as np

from .errors import DataError
from .exogenous import (ArrivalProfile, AuxSeries, CarCatalog, CatalogEntry, Dataset, PriceSeries,
                        UserScenarioModel, scenario_model)
from .physics import CarProfile
from .station import StationTree, station_from_dict, station_to_dict

__all__ = ["load_prices", "save_prices", "load_arrivals", "save_arrivals", "load_car_catalog", "save_car_catalog",
           "load_aux", "save_aux", "load_dataset", "save_dataset", "load_station", "save_station"]

TS_FORMAT = "%Y-%m-%dT%H:%M"
SCENARIO_FILE = "scenario.json"


def _rows(path: Path, required: tuple[str, ...]):
    """-> (header, [(line number, row dict)]) with the required columns checked."""
    try:
        with open(path, "r", encoding="utf-8", newline="") as fh:
            reader = csv.DictReader(fh)
            header = list(reader.fieldnames or [])
            missing = [c for c in required if c not in header]
            if missing:
                raise DataError(f"{path}: missing column(s) {', '.join(missing)}")
            rows = list(enumerate(reader, start=2))
    except OSError as exc:
        raise DataError(f"{path}: {exc}") from exc
    return header, rows


def _parse(path: Path, lineno: int, fn):
    try:
        return fn()
    except (ValueError, TypeError) as exc:
        raise DataError(f"{path}: unparseable row at line {lineno}: {exc}") from exc


def _nonempty(path: Path, rows) -> None:
    if not rows:
        raise DataError(f"{path}: no data rows")


def _write(path, header: list[str], rows) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def _hours(start: dt.date, n: int):
    t0 = dt.datetime.combine(start, dt.time())
    return [(t0 + dt.timedelta(hours=h)).strftime(TS_FORMAT) for h in range(n)]


# --- prices -------------------------------------------------------------------

def load_prices(path) -> PriceSeries:
    """Hourly price CSV; the timestamps must be contiguous whole hours."""
    path = Path(path)
    header, rows = _rows(path, ("timestamp", "buy_eur_per_kwh"))
    sell_col = "sell_grid_eur_per_kwh" if "sell_grid_eur_per_kwh" in header else "buy_eur_per_kwh"
    _nonempty(path, rows)
    buy = np.empty(len(rows))
    sell = np.empty(len(rows))
    start = None
    for h, (lineno, row) in enumerate(rows):
        ts, b, s = _parse(path, lineno, lambda: (dt.datetime.fromisoformat(row["timestamp"]),
                                                 float(row["buy_eur_per_kwh"]), float(row[sell_col])))
        if start is None:
            if ts.minute or ts.second:
                raise DataError(f"{path}: series must start on the hour (line {lineno})")
            start = ts
        want = start + dt.timedelta(hours=h)
        if ts != want:
            what = "duplicate or out-of-order hour" if ts < want else "gap"
            raise DataError(f"{path}: {what} at line {lineno}: expected {want.strftime(TS_FORMAT)}")
        buy[h], sell[h] = b, s
    return PriceSeries(start_date=start.date(), buy=buy, sell_grid=sell, region=path.stem)


def save_prices(series: PriceSeries, path) -> None:
    _write(path, ["timestamp", "buy_eur_per_kwh", "sell_grid_eur_per_kwh"],
           ([ts, repr(float(b)), repr(float(s))]
            for ts, b, s in zip(_hours(series.start_date, len(series.buy)), series.buy, series.sell_grid)))


# --- arrivals -----------------------------------------------------------------

def load_arrivals(path, weekday_scale: float = 1.0, weekend_scale: float = 1.0) -> ArrivalProfile:
    path = Path(path)
    _, rows = _rows(path, ("step_of_day", "lambda"))
    _nonempty(path, rows)
    rates = np.empty(len(rows))
    for s, (lineno, row) in enumerate(rows):
        step, lam = _parse(path, lineno, lambda: (int(row["step_of_day"]), float(row["lambda"])))
        if step != s:
            raise DataError(f"{path}: steps must be 0,1,2,... (line {lineno})")
        if lam < 0:
            raise DataError(f"{path}: negative rate at line {lineno}")
        rates[s] = lam
    return ArrivalProfile(rates_per_step=rates, weekday_scale=weekday_scale, weekend_scale=weekend_scale,
                          scenario=path.stem)


def save_arrivals(profile: ArrivalProfile, path) -> None:
    _write(path, ["step_of_day", "lambda"], ([s, repr(float(x))] for s, x in enumerate(profile.rates_per_step)))


# --- car catalogue --------------------------------------------------------------

_CAR_COLS = ("name", "capacity_kwh", "r_max_ac_kw", "r_max_dc_kw", "tau", "weight")


def load_car_catalog(path) -> CarCatalog:
    path = Path(path)
    _, rows = _rows(path, _CAR_COLS)
    _nonempty(path, rows)
    entries = []
    for lineno, row in rows:
        cap, rac, rdc, tau, w = _parse(path, lineno, lambda: tuple(float(row[c]) for c in _CAR_COLS[1:]))
        if cap <= 0:
            raise DataError(f"{path}: capacity must be positive at line {lineno}")
        if not 0.0 < tau < 1.0:
            raise DataError(f"{path}: tau must be in (0, 1) at line {lineno}")
        if w < 0:
            raise DataError(f"{path}: negative weight at line {lineno}")
        entries.append(CatalogEntry(CarProfile(capacity_kwh=cap, r_max_ac_kw=rac, r_max_dc_kw=rdc, tau=tau,
                                               name=row["name"]), w))
    if sum(e.weight for e in entries) <= 0:
        raise DataError(f"{path}: all weights are zero")
    return CarCatalog(entries=tuple(entries), region=path.stem)


def save_car_catalog(catalog: CarCatalog, path) -> None:
    _write(path, list(_CAR_COLS),
           ([e.profile.name, repr(e.profile.capacity_kwh), repr(e.profile.r_max_ac_kw), repr(e.profile.r_max_dc_kw),
             repr(e.profile.tau), repr(e.weight)] for e in catalog.entries))


# --- auxiliary series ------------------------------------------------------------

_AUX_COLS = ("moer_kg_per_kwh", "grid_demand_kwh")


def load_aux(path) -> AuxSeries:
    path = Path(path)
    header, rows = _rows(path, ("timestamp",))
    cols = [c for c in _AUX_COLS if c in header]
    if not cols:
        raise DataError(f"{path}: needs moer_kg_per_kwh and/or grid_demand_kwh")
    _nonempty(path, rows)
    vals = {c: np.empty(len(rows)) for c in cols}
    for i, (lineno, row) in enumerate(rows):
        got = _parse(path, lineno, lambda: [float(row[c]) for c in cols])
        for c, v in zip(cols, got):
            vals[c][i] = v
    return AuxSeries(moer_kg_per_kwh=vals.get("moer_kg_per_kwh"), grid_demand_kwh=vals.get("grid_demand_kwh"))


def save_aux(aux: AuxSeries, start_date: dt.date, path) -> None:
    series = [(c, getattr(aux, c)) for c in _AUX_COLS if getattr(aux, c) is not None]
    n = max((len(v) for _, v in series), default=0)
    _write(path, ["timestamp"] + [c for c, _ in series],
           ([ts] + [repr(float(v[h])) for _, v in series] for h, ts in enumerate(_hours(start_date, n))))


# --- dataset directory ---------------------------------------------------------------

def load_dataset(data_dir, weekday_scale: float | None = None, weekend_scale: float | None = None) -> Dataset:
    """prices/arrivals/cars CSVs + optional aux.csv and scenario.json."""
    d = Path(data_dir)
    meta = {}
    if (d / SCENARIO_FILE).exists():
        try:
            meta = json.loads((d / SCENARIO_FILE).read_text(encoding="utf-8"))
        except (OSError, json.JSONDecodeError) as exc:
            raise DataError(f"{d / SCENARIO_FILE}: {exc}") from exc
    wk = float(meta.get("weekday_scale", 1.0)) if weekday_scale is None else weekday_scale
    we = float(meta.get("weekend_scale", 1.0)) if weekend_scale is None else weekend_scale
    if "stay_steps_range" in meta:
        scen = UserScenarioModel(stay_steps_range=tuple(meta["stay_steps_range"]),
                                 requested_fraction_range=tuple(meta["requested_fraction_range"]),
                                 soc_arrival_range=tuple(meta["soc_arrival_range"]),
                                 p_charge_sensitive=float(meta["p_charge_sensitive"]),
                                 scenario=str(meta.get("scenario", "custom")))
    else:
        scen = scenario_model(meta.get("scenario", "shopping"))
    aux = load_aux(d / "aux.csv") if (d / "aux.csv").exists() else AuxSeries()
    return Dataset(prices=load_prices(d / "prices.csv"),
                   arrivals=load_arrivals(d / "arrivals.csv", weekday_scale=wk, weekend_scale=we),
                   cars=load_car_catalog(d / "cars.csv"), scenario=scen, aux=aux)


def save_dataset(ds: Dataset, data_dir) -> None:
    d = Path(data_dir)
    d.mkdir(parents=True, exist_ok=True)
    save_prices(ds.prices, d / "prices.csv")
    save_arrivals(ds.arrivals, d / "arrivals.csv")
    save_car_catalog(ds.cars, d / "cars.csv")
    if ds.aux.moer_kg_per_kwh is not None or ds.aux.grid_demand_kwh is not None:
        save_aux(ds.aux, ds.prices.start_date, d / "aux.csv")
    s = ds.scenario
    meta = {"scenario": s.scenario, "stay_steps_range": list(s.stay_steps_range),
            "requested_fraction_range": list(s.requested_fraction_range),
            "soc_arrival_range": list(s.soc_arrival_range), "p_charge_sensitive": s.p_charge_sensitive,
            "weekday_scale": ds.arrivals.weekday_scale, "weekend_scale": ds.arrivals.weekend_scale}
    (d / SCENARIO_FILE).write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n", encoding="utf-8")


# --- station JSON ---------------------------------------------------------------------

def load_station(path) -> StationTree:
    """Nested-node station JSON (topology.py:452-500)."""
    with open(path, "r", encoding="utf-8") as fh:
        return station_from_dict(json.load(fh))


def save_station(tree: StationTree, path) -> None:
    Path(path).write_text(json.dumps(station_to_dict(tree), indent=2, sort_keys=True) + "\n", encoding="utf-8")
