"""Flatten (config, station, dataset) into the read-only step tables.

Mirror of ``build_tables`` (``voltyard/engine.py:107-218``): same content,
same dtypes for the float64 data, int32 for indices.  The result feeds the
C-ABI (``vy_tables`` in include/voltyard_b200.h) of both the CUDA library and
the CPU oracle, so both sides step from byte-identical tables.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, fields

import numpy as np

from .envconfig import DEFAULT_BATTERY, EnvConfig, ObsLayout
from .errors import DataError
from .exogenous import Dataset
from .physics import BatterySpec
from .station import StationTree, compile_tree

_F64 = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I8 = C.POINTER(C.c_int8)


class VyTables(C.Structure):
    """ctypes twin of ``vy_tables`` (include/voltyard_b200.h)."""

    _fields_ = [
        ("n_ports", C.c_int32), ("n_slots", C.c_int32), ("n_nodes", C.c_int32), ("max_passes", C.c_int32),
        ("volt", _F64), ("imax_c", _F64), ("imax_d", _F64), ("eta_c", _F64), ("eta_d", _F64), ("i_denom", _F64),
        ("kind", _I32), ("order", _I32),
        ("node_cap", _F64), ("node_eta", _F64),
        ("node_ptr", _I32), ("node_leaf", _I32), ("node_order", _I32),
        ("battery_enabled", C.c_int32),
        ("b_volt", C.c_double), ("b_cap", C.c_double), ("b_rmax", C.c_double), ("b_tau", C.c_double),
        ("b_eta_c", C.c_double), ("b_eta_d", C.c_double), ("b_init_soc", C.c_double),
        ("b_imax", C.c_double), ("b_idenom", C.c_double),
        ("k", C.c_int32), ("episode_steps", C.c_int32), ("steps_per_day", C.c_int32), ("dt_min", C.c_int32),
        ("horizon", C.c_int32), ("obs_len", C.c_int32), ("allow_discharge", C.c_int32),
        ("dt_h", C.c_double), ("p_sell", C.c_double), ("c_dt", C.c_double), ("beta", C.c_double),
        ("alphas", C.c_double * 8),
        ("n_days", C.c_int32), ("lam_len", C.c_int32), ("has_moer", C.c_int32), ("has_dgrid", C.c_int32),
        ("wk_scale", C.c_double), ("we_scale", C.c_double),
        ("buy", _F64), ("sellg", _F64), ("lam", _F64), ("weekday", _I8),
        ("moer", _F64), ("dgrid", _F64), ("sin_t", _F64), ("cos_t", _F64),
        ("n_cat", C.c_int32), ("stay_lo", C.c_int32), ("stay_hi", C.c_int32),
        ("cat_cum", _F64), ("cat_cap", _F64), ("cat_rac", _F64), ("cat_rdc", _F64), ("cat_tau", _F64),
        ("soc_lo", C.c_double), ("soc_hi", C.c_double), ("frac_lo", C.c_double), ("frac_hi", C.c_double),
        ("p_charge", C.c_double),
    ]


@dataclass
class StepTables:
    """Read-only inputs shared by every env of a batch (KernelTables twin)."""

    n_ports: int
    n_slots: int
    volt: np.ndarray
    imax_c: np.ndarray
    imax_d: np.ndarray
    eta_c: np.ndarray
    eta_d: np.ndarray
    i_denom: np.ndarray
    kind: np.ndarray
    order: np.ndarray
    n_nodes: int
    node_cap: np.ndarray
    node_eta: np.ndarray
    node_ptr: np.ndarray
    node_leaf: np.ndarray
    node_order: np.ndarray
    max_passes: int
    battery_enabled: bool
    b_volt: float
    b_cap: float
    b_rmax: float
    b_tau: float
    b_eta_c: float
    b_eta_d: float
    b_init_soc: float
    b_imax: float
    b_idenom: float
    k: int
    episode_steps: int
    steps_per_day: int
    dt_min: int
    dt_h: float
    p_sell: float
    c_dt: float
    beta: float
    alphas: np.ndarray
    allow_discharge: bool
    horizon: int
    obs_len: int
    n_days: int
    buy: np.ndarray
    sellg: np.ndarray
    lam: np.ndarray
    lam_len: int
    wk_scale: float
    we_scale: float
    weekday: np.ndarray
    has_moer: bool
    moer: np.ndarray
    has_dgrid: bool
    dgrid: np.ndarray
    sin_t: np.ndarray
    cos_t: np.ndarray
    n_cat: int
    cat_cum: np.ndarray
    cat_cap: np.ndarray
    cat_rac: np.ndarray
    cat_rdc: np.ndarray
    cat_tau: np.ndarray
    stay_lo: int
    stay_hi: int
    soc_lo: float
    soc_hi: float
    frac_lo: float
    frac_hi: float
    p_charge: float

    _ct: VyTables | None = None

    def as_ctypes(self) -> VyTables:
        """The vy_tables struct; pointers alias this object's contiguous arrays."""
        if self._ct is not None:
            return self._ct
        ct = VyTables()
        for f in VyTables._fields_:
            name, typ = f
            val = getattr(self, name)
            if isinstance(val, np.ndarray) and name != "alphas":
                want = {_F64: np.float64, _I32: np.int32, _I8: np.int8}[typ]
                arr = np.ascontiguousarray(val, dtype=want)
                setattr(self, name, arr)
                setattr(ct, name, arr.ctypes.data_as(typ))
            elif name == "alphas":
                for i in range(8):
                    ct.alphas[i] = float(self.alphas[i])
            else:
                setattr(ct, name, int(val) if typ is C.c_int32 else float(val))
        self._ct = ct
        return ct

    def hour_series(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self) if isinstance(getattr(self, f.name), np.ndarray)}


def _tile_hourly(series, present: bool, n_hours: int) -> np.ndarray:
    """engine.py:137-145: aux series clipped or tiled to the price range."""
    if not present:
        return np.zeros(1)
    s = np.asarray(series, dtype=np.float64)
    if len(s) >= n_hours:
        return s[:n_hours].copy()
    return np.tile(s, -(-n_hours // len(s)))[:n_hours]


def build_tables(config: EnvConfig, station: StationTree, dataset: Dataset) -> StepTables:
    ev = station.evses
    n = len(ev)
    tree = compile_tree(station, include_battery=config.battery_enabled)
    batt = station.battery
    if config.battery_enabled and batt is None:
        batt = DEFAULT_BATTERY
    if batt is None:
        batt = BatterySpec(voltage_v=1.0, capacity_kwh=1.0, r_max_kw=0.0, tau=0.5)
    if dataset.prices.n_days < 1:
        raise DataError("dataset must cover at least one day")
    imax_c = np.array([e.i_max_charge_a for e in ev], dtype=np.float64)
    imax_d = np.array([e.i_max_discharge_a for e in ev], dtype=np.float64)
    spd = config.steps_per_day
    ang = 2.0 * math.pi * np.arange(spd) / spd
    n_hours = len(dataset.prices.buy)
    aux = dataset.aux
    b_imax = 1000.0 * batt.r_max_kw / batt.voltage_v
    scen = dataset.scenario
    return StepTables(
        n_ports=n, n_slots=tree.n_slots,
        volt=np.array([e.voltage_v for e in ev], dtype=np.float64),
        imax_c=imax_c, imax_d=imax_d,
        eta_c=np.array([e.eta_charge for e in ev], dtype=np.float64),
        eta_d=np.array([e.eta_discharge for e in ev], dtype=np.float64),
        i_denom=np.where(imax_c > 0, imax_c, np.where(imax_d > 0, imax_d, 1.0)).astype(np.float64),
        kind=np.array([1 if e.kind == "dc" else 0 for e in ev], dtype=np.int32),
        order=np.asarray(station.parking_order, dtype=np.int32),
        n_nodes=len(tree.node_cap), node_cap=tree.node_cap, node_eta=tree.node_eta,
        node_ptr=tree.node_ptr.astype(np.int32), node_leaf=tree.node_leaf.astype(np.int32),
        node_order=tree.order_desc.astype(np.int32), max_passes=2 * tree.depth + 4,
        battery_enabled=bool(config.battery_enabled),
        b_volt=float(batt.voltage_v), b_cap=float(batt.capacity_kwh), b_rmax=float(batt.r_max_kw),
        b_tau=float(batt.tau), b_eta_c=float(batt.eta_charge), b_eta_d=float(batt.eta_discharge),
        b_init_soc=float(config.battery_init_soc), b_imax=b_imax,
        b_idenom=b_imax if (config.battery_enabled and b_imax > 0) else 1.0,
        k=config.discretization_k, episode_steps=config.episode_steps, steps_per_day=spd,
        dt_min=config.dt_min, dt_h=config.dt_hours, p_sell=float(config.p_sell_eur_per_kwh),
        c_dt=float(config.fixed_cost_per_step), beta=float(config.beta), alphas=config.alpha_array(),
        allow_discharge=bool(config.allow_discharge), horizon=config.observe_price_horizon,
        obs_len=ObsLayout(n_ports=n, horizon=config.observe_price_horizon).length,
        n_days=dataset.prices.n_days,
        buy=np.asarray(dataset.prices.buy, dtype=np.float64),
        sellg=np.asarray(dataset.prices.sell_grid, dtype=np.float64),
        lam=np.asarray(dataset.arrivals.rates_per_step, dtype=np.float64),
        lam_len=len(dataset.arrivals.rates_per_step),
        wk_scale=float(dataset.arrivals.weekday_scale), we_scale=float(dataset.arrivals.weekend_scale),
        weekday=dataset.prices.weekday_mask(),
        has_moer=aux.moer_kg_per_kwh is not None,
        moer=_tile_hourly(aux.moer_kg_per_kwh, aux.moer_kg_per_kwh is not None, n_hours),
        has_dgrid=aux.grid_demand_kwh is not None,
        dgrid=_tile_hourly(aux.grid_demand_kwh, aux.grid_demand_kwh is not None, n_hours),
        sin_t=np.sin(ang), cos_t=np.cos(ang),
        n_cat=len(dataset.cars.entries), cat_cum=dataset.cars.cumulative_weights(),
        cat_cap=np.array([e.profile.capacity_kwh for e in dataset.cars.entries], dtype=np.float64),
        cat_rac=np.array([e.profile.r_max_ac_kw for e in dataset.cars.entries], dtype=np.float64),
        cat_rdc=np.array([e.profile.r_max_dc_kw for e in dataset.cars.entries], dtype=np.float64),
        cat_tau=np.array([e.profile.tau for e in dataset.cars.entries], dtype=np.float64),
        stay_lo=int(scen.stay_steps_range[0]), stay_hi=int(scen.stay_steps_range[1]),
        soc_lo=float(scen.soc_arrival_range[0]), soc_hi=float(scen.soc_arrival_range[1]),
        frac_lo=float(scen.requested_fraction_range[0]), frac_hi=float(scen.requested_fraction_range[1]),
        p_charge=float(scen.p_charge_sensitive),
    )


def build_tables_from_kernel_tables(kt) -> StepTables:
    """StepTables from any object with the reference KernelTables fields
    (engine.py:30-104), e.g. the reference engine's own ``env.tables``."""
    names = [f.name for f in fields(StepTables) if not f.name.startswith("_")]
    return StepTables(**{n: getattr(kt, n) for n in names})
