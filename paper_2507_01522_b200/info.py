"""Per-step info records decoded from the device info block.

Types mirror ``voltyard/env.py:22-105``; ``step_infos`` is the batched
counterpart of ``step_info_from_outputs`` (env.py:108-154): one D2H copy of
the feature-major info block, then per-env records on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RewardBreakdown:
    profit_eur: float
    c_constraint: float
    c_sat0: float
    c_sat1: float
    c_sustain: float
    c_declined: float
    c_degrad_battery: float
    c_degrad_cars: float
    c_grid: float
    total: float

    def penalties(self) -> dict:
        return {"constraint": self.c_constraint, "sat0": self.c_sat0, "sat1": self.c_sat1,
                "sustain": self.c_sustain, "declined": self.c_declined,
                "degrad_battery": self.c_degrad_battery, "degrad_cars": self.c_degrad_cars, "grid": self.c_grid}


@dataclass(frozen=True)
class EnergyFlows:
    e_net: float
    e_grid_in: float
    e_to_grid: float
    e_battery_net: float
    e_grid_net: float


@dataclass(frozen=True)
class Departure:
    port: int
    preference: int
    missing_kwh: float
    overtime_steps: int
    early_steps: int
    capacity_kwh: float
    soc_final: float


@dataclass(frozen=True)
class EpisodeStats:
    profit_eur: float
    reward: float
    missing_kwh: float
    overtime_steps: int
    declined: int
    energy_net_kwh: float
    departures: int
    terminal_overtime_steps: int


@dataclass(frozen=True)
class StepInfo:
    flows: EnergyFlows
    breakdown: RewardBreakdown
    departures: tuple
    declined: int
    arrivals_sampled: int
    done: bool
    episode: EpisodeStats | None
    currents_attempted_a: np.ndarray
    currents_applied_a: np.ndarray
    delivered_kwh: np.ndarray
    battery_delivered_kwh: float


def step_infos(env) -> list:
    o = env.reference_outputs()
    done = env.outs.done.cpu().numpy().astype(bool)
    out = []
    for b in range(env.batch_size):
        br = o["breakdown"][b]
        fl = o["flows"][b]
        deps = tuple(
            Departure(int(o["dep_port"][b, j]), int(o["dep_pref"][b, j]), float(o["dep_missing"][b, j]),
                      int(o["dep_overtime"][b, j]), int(o["dep_early"][b, j]), float(o["dep_cap"][b, j]),
                      float(o["dep_soc"][b, j]))
            for j in range(int(o["dep_n"][b])))
        ep = None
        if done[b]:
            es = o["ep_stats"][b]
            ep = EpisodeStats(es[0], es[1], es[2], int(es[3]), int(es[4]), es[5], int(es[6]), int(es[7]))
        out.append(StepInfo(
            flows=EnergyFlows(*fl[:5]), breakdown=RewardBreakdown(*br[:10]), departures=deps,
            declined=int(o["declined"][b]), arrivals_sampled=int(o["arrivals_m"][b]), done=bool(done[b]),
            episode=ep, currents_attempted_a=o["i_att"][b].copy(), currents_applied_a=o["i_used"][b].copy(),
            delivered_kwh=o["delivered"][b].copy(), battery_delivered_kwh=float(o["b_delivered"][b])))
    return out
