"""Exogenous inputs: prices, arrival rates, car catalogue, user scenarios.

Host-side mirror of ``voltyard/data.py`` (types data.py:40-183, samplers
:188-261, synthetic generators :532-672).  These are table *producers*: the
device consumes their flattened form (``tables.py``).  The synthetic
generators must reproduce the reference's arrays bit for bit (same draw
order, same libm calls, same float expression trees) because the parity
tests feed identical tables to the CUDA kernels and the CPU oracle;
``tests/test_host_mirror.py`` pins them against committed golden arrays.
"""

from __future__ import annotations

import datetime as dt
import math
from dataclasses import dataclass, field

import numpy as np

from .errors import DataError
from .physics import CarProfile, UserProfile
from .streams import BatchStreams, Stream, stream_key

SCENARIOS = ("highway", "residential", "work", "shopping")
TRAFFIC_FACTORS = {"low": 0.5, "medium": 1.0, "high": 2.0}
REGIONS = ("eu", "us", "world")


@dataclass(frozen=True)
class PriceSeries:
    """Hourly buy and grid sell-back prices (EUR/kWh), whole days."""

    start_date: dt.date
    buy: np.ndarray
    sell_grid: np.ndarray
    region: str = ""

    def __post_init__(self):
        b = np.asarray(self.buy, dtype=np.float64)
        s = np.asarray(self.sell_grid, dtype=np.float64)
        object.__setattr__(self, "buy", b)
        object.__setattr__(self, "sell_grid", s)
        if b.shape != s.shape:
            raise DataError("buy and sell_grid series must have equal length")
        if len(b) == 0 or len(b) % 24:
            raise DataError(f"price series length must be a positive multiple of 24, got {len(b)}")
        if not (np.isfinite(b).all() and np.isfinite(s).all()):
            raise DataError("price series contains non-finite values")

    @property
    def n_days(self) -> int:
        return len(self.buy) // 24

    def is_weekday(self, day: int) -> bool:
        return (self.start_date + dt.timedelta(days=day)).weekday() < 5

    def weekday_mask(self) -> np.ndarray:
        return np.array([self.is_weekday(d) for d in range(self.n_days)], dtype=np.int8)


@dataclass(frozen=True)
class ArrivalProfile:
    """Mean arrivals per step of day, with weekday / weekend multipliers."""

    rates_per_step: np.ndarray
    weekday_scale: float = 1.0
    weekend_scale: float = 1.0
    scenario: str = ""

    def __post_init__(self):
        r = np.asarray(self.rates_per_step, dtype=np.float64)
        object.__setattr__(self, "rates_per_step", r)
        if len(r) == 0:
            raise DataError("arrival profile is empty")
        if not np.isfinite(r).all() or (r < 0).any():
            raise DataError("arrival rates must be finite and >= 0")
        if self.weekday_scale < 0 or self.weekend_scale < 0:
            raise DataError("arrival scales must be >= 0")


@dataclass(frozen=True)
class CatalogEntry:
    profile: CarProfile
    weight: float


@dataclass(frozen=True)
class CarCatalog:
    entries: tuple
    region: str = ""

    def __post_init__(self):
        if not self.entries:
            raise DataError("car catalog is empty")
        if any(e.weight < 0 for e in self.entries):
            raise DataError("negative catalog weight")
        if sum(e.weight for e in self.entries) <= 0:
            raise DataError("car catalog weights sum to zero")

    def cumulative_weights(self) -> np.ndarray:
        w = np.array([e.weight for e in self.entries], dtype=np.float64)
        return np.cumsum(w / w.sum())


@dataclass(frozen=True)
class UserScenarioModel:
    stay_steps_range: tuple
    requested_fraction_range: tuple
    soc_arrival_range: tuple
    p_charge_sensitive: float
    scenario: str = ""

    def __post_init__(self):
        lo, hi = self.stay_steps_range
        if not 1 <= lo <= hi:
            raise DataError("stay_steps_range must satisfy 1 <= lo <= hi")
        for nm in ("requested_fraction_range", "soc_arrival_range"):
            a, b = getattr(self, nm)
            if not 0.0 <= a <= b <= 1.0:
                raise DataError(f"{nm} must be ordered within (0.0, 1.0)")
        if not 0.0 <= self.p_charge_sensitive <= 1.0:
            raise DataError("p_charge_sensitive must be in [0, 1]")


@dataclass(frozen=True)
class AuxSeries:
    moer_kg_per_kwh: np.ndarray | None = None
    grid_demand_kwh: np.ndarray | None = None


@dataclass(frozen=True)
class ExogenousFrame:
    p_buy: float
    p_sell_grid: float
    lambda_arrivals: float
    moer_kg_per_kwh: float | None
    grid_demand_kwh: float | None
    day_index: int
    is_weekday: bool
    step_of_day: int


@dataclass(frozen=True)
class Dataset:
    prices: PriceSeries
    arrivals: ArrivalProfile
    cars: CarCatalog
    scenario: UserScenarioModel
    aux: AuxSeries = field(default_factory=AuxSeries)

    def meta(self) -> dict:
        return {
            "price_region": self.prices.region,
            "days": self.prices.n_days,
            "start_date": self.prices.start_date.isoformat(),
            "arrival_scenario": self.arrivals.scenario,
            "car_region": self.cars.region,
            "user_scenario": self.scenario.scenario,
            "has_moer": self.aux.moer_kg_per_kwh is not None,
            "has_grid_demand": self.aux.grid_demand_kwh is not None,
        }


# --- samplers: the draw order the kernels replay (data.py:188-219) ----------

def sample_arrival_count(stream: Stream, lam: float) -> int:
    if lam < 0:
        raise ValueError(f"arrival rate must be >= 0, got {lam}")
    return stream.poisson(lam)


def sample_car(stream: Stream, catalog: CarCatalog) -> CarProfile:
    return catalog.entries[stream.choice_cum(catalog.cumulative_weights())].profile


def sample_user(stream: Stream, model: UserScenarioModel, car: CarProfile) -> UserProfile:
    """Draws in fixed order: stay, soc, fraction, preference."""
    lo, hi = model.stay_steps_range
    stay = lo + stream.randint(hi - lo + 1)
    s_lo, s_hi = model.soc_arrival_range
    soc0 = s_lo + stream.uniform() * (s_hi - s_lo)
    f_lo, f_hi = model.requested_fraction_range
    frac = f_lo + stream.uniform() * (f_hi - f_lo)
    pref = 1 if stream.uniform() < model.p_charge_sensitive else 0
    return UserProfile(stay_steps=stay, energy_requested_kwh=frac * car.capacity_kwh * (1.0 - soc0),
                       soc_arrival=soc0, preference=pref)


def frame_at(prices: PriceSeries, arrivals: ArrivalProfile, aux: AuxSeries | None,
             day: int, step: int, dt_min: int) -> ExogenousFrame:
    """Signals at (day, step) with hourly zero-order hold (data.py:222-261)."""
    minutes = step * dt_min
    eff = day + minutes // 1440
    if not 0 <= day < prices.n_days or eff >= prices.n_days:
        raise DataError(f"day {eff} outside loaded range of {prices.n_days} days")
    h = eff * 24 + (minutes // 60) % 24
    spd = len(arrivals.rates_per_step)
    wk = prices.is_weekday(eff)
    lam = float(arrivals.rates_per_step[step % spd]) * (arrivals.weekday_scale if wk else arrivals.weekend_scale)

    def hold(series):
        return None if series is None else float(series[h % len(series)])

    aux = aux or AuxSeries()
    return ExogenousFrame(float(prices.buy[h]), float(prices.sell_grid[h]), lam,
                          hold(aux.moer_kg_per_kwh), hold(aux.grid_demand_kwh),
                          eff, wk, step % spd)


# --- synthetic stand-in data (data.py:532-672) ------------------------------

_MARKETS = {"nl": (0.11, 0.07, 0.012), "fr": (0.10, 0.05, 0.010), "de": (0.12, 0.08, 0.014)}
_REGION_MARKET = {"eu": "nl", "us": "fr", "world": "de"}
_DAILY_ARRIVALS = 60.0
_DAY_SCALES = {"highway": (1.0, 1.2), "residential": (1.0, 1.1), "work": (1.0, 0.3), "shopping": (1.0, 1.3)}
# stay (minutes), requested fraction, arrival soc, P(charge-sensitive)
_SCENARIO = {
    "highway": ((15, 60), (0.4, 0.9), (0.1, 0.5), 0.7),
    "residential": ((480, 840), (0.5, 1.0), (0.2, 0.6), 0.1),
    "work": ((420, 570), (0.3, 0.9), (0.3, 0.7), 0.05),
    "shopping": ((45, 180), (0.2, 0.8), (0.3, 0.8), 0.3),
}
# name, capacity kWh, AC kW, DC kW, tau, weight
_CARS = {
    "eu": (("compact", 40.0, 7.4, 60.0, 0.80, 0.35), ("midsize", 62.0, 11.0, 120.0, 0.80, 0.45),
           ("executive", 90.0, 11.0, 180.0, 0.85, 0.20)),
    "us": (("crossover", 75.0, 9.6, 120.0, 0.80, 0.50), ("pickup", 130.0, 11.5, 190.0, 0.85, 0.30),
           ("sedan", 100.0, 11.5, 250.0, 0.85, 0.20)),
    "world": (("city", 30.0, 6.6, 50.0, 0.80, 0.30), ("compact", 45.0, 7.4, 80.0, 0.80, 0.30),
              ("midsize", 62.0, 11.0, 120.0, 0.80, 0.25), ("executive", 95.0, 11.0, 200.0, 0.85, 0.15)),
}


def _bump(x: float, centre: float, width: float) -> float:
    return math.exp(-(((x - centre) / width) ** 2))


def _arrival_shape(scenario: str, hour: float) -> float:
    if scenario == "shopping":
        return 0.05 + _bump(hour, 13.5, 2.5)
    if scenario == "work":
        return 0.03 + _bump(hour, 8.5, 1.5) + 0.3 * _bump(hour, 13.0, 2.0)
    if scenario == "residential":
        return 0.08 + _bump(hour, 19.0, 2.5) + 0.3 * _bump(hour, 7.5, 1.5)
    return 0.6 + 0.4 * _bump(hour, 14.0, 6.0)


def scenario_model(scenario: str, dt_min: int = 5) -> UserScenarioModel:
    if scenario not in SCENARIOS:
        raise DataError(f"unknown scenario {scenario!r}; pick one of {SCENARIOS}")
    (lo, hi), frac, soc, pc = _SCENARIO[scenario]
    return UserScenarioModel((max(1, round(lo / dt_min)), max(1, round(hi / dt_min))),
                             frac, soc, pc, scenario)


def car_catalog(region: str) -> CarCatalog:
    if region not in REGIONS:
        raise DataError(f"unknown region {region!r}; pick one of {REGIONS}")
    return CarCatalog(tuple(CatalogEntry(CarProfile(c, ac, dc, tau, name=n), w)
                            for n, c, ac, dc, tau, w in _CARS[region]), region=region)


def _unit_draws(key: int, n: int) -> np.ndarray:
    """First n uniforms of stream ``key`` in one vectorised pass."""
    return BatchStreams(np.array([key], dtype=np.uint64)).uniform_block(n)[0]


def synthetic_prices(region: str = "eu", seed: int = 0, days: int = 365) -> PriceSeries:
    market = _REGION_MARKET.get(region, region)
    if market not in _MARKETS:
        raise DataError(f"unknown price region {region!r}")
    base, amp, noise = _MARKETS[market]
    hourly = np.array([_bump(h, 8.0, 3.0) + _bump(h, 19.0, 3.0) for h in range(24)])
    shape = np.tile(hourly, days)
    u = _unit_draws(stream_key(seed, 101), days * 24)
    buy = base + amp * (shape - 0.5) + noise * (2.0 * u - 1.0)
    return PriceSeries(dt.date(2022, 1, 3), buy, buy - 0.01, region=market)


def synthetic_arrivals(scenario: str = "shopping", traffic: str = "medium", dt_min: int = 5) -> ArrivalProfile:
    if traffic not in TRAFFIC_FACTORS:
        raise DataError(f"unknown traffic level {traffic!r}; pick one of {tuple(TRAFFIC_FACTORS)}")
    if scenario not in SCENARIOS:
        raise DataError(f"unknown scenario {scenario!r}; pick one of {SCENARIOS}")
    shape = np.array([_arrival_shape(scenario, s * dt_min / 60.0) for s in range(1440 // dt_min)])
    curve = _DAILY_ARRIVALS * shape / shape.sum()
    wk, we = _DAY_SCALES[scenario]
    return ArrivalProfile(TRAFFIC_FACTORS[traffic] * curve, wk, we, f"{scenario}-{traffic}")


def synthetic_aux(seed: int = 0, days: int = 365) -> AuxSeries:
    n = days * 24
    u = _unit_draws(stream_key(seed, 202), 2 * n).reshape(n, 2)
    hod = (np.arange(n) % 24).astype(np.float64)
    sin_m = np.array([math.sin(2.0 * math.pi * (h - 4.0) / 24.0) for h in range(24)])
    sin_d = np.array([math.sin(2.0 * math.pi * (h - 10.0) / 24.0) for h in range(24)])
    idx = hod.astype(np.int64)
    moer = 0.30 + 0.12 * sin_m[idx] + 0.02 * (2.0 * u[:, 0] - 1.0)
    demand = 20.0 + 15.0 * sin_d[idx] + 2.0 * (2.0 * u[:, 1] - 1.0)
    return AuxSeries(moer, demand)


def generate_synthetic_defaults(scenario: str = "shopping", traffic: str = "medium", region: str = "eu",
                                seed: int = 0, days: int = 365, dt_min: int = 5,
                                with_aux: bool = False) -> Dataset:
    return Dataset(
        prices=synthetic_prices(region=region, seed=seed, days=days),
        arrivals=synthetic_arrivals(scenario=scenario, traffic=traffic, dt_min=dt_min),
        cars=car_catalog(region),
        scenario=scenario_model(scenario, dt_min=dt_min),
        aux=synthetic_aux(seed=seed, days=days) if with_aux else AuxSeries(),
    )
