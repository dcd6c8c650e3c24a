"""Environment configuration, penalty order and observation layout.

Mirror of ``voltyard/config.py`` (``PENALTY_NAMES`` :19-28, ``DEFAULT_BATTERY``
:30, ``EnvConfig`` :33-96, ``ObsLayout`` :99-130, ``default_setup`` :226-245).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import exogenous, station
from .physics import BatterySpec

# the reward subtracts alpha_c * c_c in exactly this order
PENALTY_NAMES = (
    "constraint", "sat0", "sat1", "sustain", "declined", "degrad_battery", "degrad_cars", "grid",
)

DEFAULT_BATTERY = BatterySpec(voltage_v=800.0, capacity_kwh=200.0, r_max_kw=100.0, tau=0.8)


@dataclass
class EnvConfig:
    dt_min: int = 5
    episode_steps: int = 288
    discretization_k: int = 10
    p_sell_eur_per_kwh: float = 0.75
    fixed_cost_per_step: float = 0.0
    alpha: dict = field(default_factory=dict)
    beta: float = 0.0
    allow_discharge: bool = True
    battery_enabled: bool = False
    battery_init_soc: float = 0.5
    observe_price_horizon: int = 0

    def __post_init__(self):
        if self.dt_min <= 0 or 1440 % self.dt_min:
            raise ValueError("dt_min must be positive and divide 1440")
        if self.episode_steps < 1:
            raise ValueError("episode_steps must be >= 1")
        if self.discretization_k < 1:
            raise ValueError("discretization_k must be >= 1")
        if not 0.0 <= self.battery_init_soc <= 1.0:
            raise ValueError("battery_init_soc must be in [0, 1]")
        if self.observe_price_horizon < 0:
            raise ValueError("observe_price_horizon must be >= 0")
        bad = sorted(set(self.alpha) - set(PENALTY_NAMES))
        if bad:
            raise ValueError(f"unknown penalty name(s) {bad}; valid: {PENALTY_NAMES}")

    def alpha_array(self) -> np.ndarray:
        return np.array([float(self.alpha.get(n, 0.0)) for n in PENALTY_NAMES])

    @property
    def dt_hours(self) -> float:
        return self.dt_min / 60.0

    @property
    def steps_per_day(self) -> int:
        return 1440 // self.dt_min

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d["alpha"] = {k: float(v) for k, v in sorted(self.alpha.items())}
        return d

    @classmethod
    def from_dict(cls, obj: dict) -> "EnvConfig":
        return cls(**obj)


@dataclass(frozen=True)
class ObsLayout:
    """Per port [occ, I/Imax, soc, de/C, dtrem/T, pref]; battery [soc, I/Imax];
    globals [p_buy, p_sell_grid, p_sell, sin, cos, weekday, day/365]; horizon."""

    n_ports: int
    horizon: int
    per_port: int = 6

    @property
    def battery_offset(self) -> int:
        return self.per_port * self.n_ports

    @property
    def globals_offset(self) -> int:
        return self.battery_offset + 2

    @property
    def horizon_offset(self) -> int:
        return self.globals_offset + 7

    @property
    def length(self) -> int:
        return self.horizon_offset + self.horizon

    def port_offset(self, i: int) -> int:
        return self.per_port * i


@dataclass
class RunConfig:
    env: EnvConfig
    station: station.StationTree
    dataset: exogenous.Dataset


def default_setup(env: EnvConfig | None = None, scenario: str = "shopping", traffic: str = "medium",
                  region: str = "eu", seed: int = 0, days: int = 365, with_aux: bool = False) -> RunConfig:
    """The reference 16-port station on synthetic data."""
    env = env if env is not None else EnvConfig()
    return RunConfig(
        env=env,
        station=station.default_station(battery=DEFAULT_BATTERY if env.battery_enabled else None),
        dataset=exogenous.generate_synthetic_defaults(scenario=scenario, traffic=traffic, region=region,
                                                      seed=seed, days=days, dt_min=env.dt_min,
                                                      with_aux=with_aux),
    )
