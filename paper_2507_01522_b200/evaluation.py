"""Paired-seed policy evaluation on the device (reference evaluate.py:23-142).

Episode j runs env seed split_seed(seed, j) with auto-reset off for exactly
episode_steps steps; its ep_stats row (written in-kernel at episode end) is
the per-episode record.  The reference evaluates in chunks of 128 envs
(evaluate.py:20, 96-104); envs are independent, so one batch of all episodes
gives the identical records.
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from .batch import BatchEnv
from .envconfig import EnvConfig
from .exogenous import Dataset
from .station import StationTree, station_to_dict
from .streams import split_seed


def fingerprint(config: EnvConfig, station: StationTree, dataset: Dataset) -> str:
    """config.py:133-143."""
    blob = json.dumps({"config": config.to_dict(), "station": station_to_dict(station), "dataset": dataset.meta()},
                      sort_keys=True).encode()
    return hashlib.sha256(blob).hexdigest()[:16]


def _r9(x: float) -> float:
    if x == 0 or not math.isfinite(x):
        return float(x)
    return float(f"{x:.9g}")


@dataclass(frozen=True)
class MetricsReport:
    mean_daily_profit_eur: float
    std_daily_profit_eur: float
    mean_reward: float
    missing_kwh_per_departure: float
    overtime_steps_per_departure: float
    declined_per_episode: float
    energy_sold_kwh_per_episode: float
    episodes: int
    config_fingerprint: str
    per_episode: tuple

    def to_dict(self) -> dict:
        d = {k: (_r9(v) if isinstance(v, float) else v) for k, v in self.__dict__.items() if k != "per_episode"}
        d["per_episode"] = [{k: (_r9(v) if isinstance(v, float) else v) for k, v in ep.items()}
                            for ep in self.per_episode]
        return d


_FIELDS = ("profit_eur", "reward", "missing_kwh", "overtime_steps", "declined", "energy_net_kwh", "departures",
           "terminal_overtime_steps")
_INT = {"overtime_steps", "declined", "departures", "terminal_overtime_steps"}


def evaluate(policy, config: EnvConfig, station: StationTree, dataset: Dataset, episodes: int = 1, seed: int = 0,
             backend: str | None = None) -> MetricsReport:
    if episodes < 1:
        raise ValueError("episodes must be >= 1")
    env = BatchEnv(config, station, dataset, batch_size=episodes,
                   env_seeds=[split_seed(seed, j) for j in range(episodes)], auto_reset=False, backend=backend,
                   obs_dtype=torch.float64)
    policy.bind(range(episodes))
    obs = env.reset(as_numpy=False)
    for _ in range(config.episode_steps):
        obs, _, _, _ = env.step(policy.actions(obs, env), collect_infos=False)
    es = env.outs.ep_stats[:, :episodes].T.cpu().numpy()
    env.close()
    records = []
    for j in range(episodes):
        rec = {"episode": j}
        for i, f in enumerate(_FIELDS):
            rec[f] = int(es[j, i]) if f in _INT else float(es[j, i])
        records.append(rec)
    profits = np.array([r["profit_eur"] for r in records])
    rewards = np.array([r["reward"] for r in records])
    departures = sum(r["departures"] for r in records)
    missing = sum(r["missing_kwh"] for r in records)
    overtime = sum(r["overtime_steps"] for r in records)
    return MetricsReport(
        mean_daily_profit_eur=float(profits.mean()),
        std_daily_profit_eur=float(profits.std(ddof=1)) if episodes > 1 else 0.0,
        mean_reward=float(rewards.mean()),
        missing_kwh_per_departure=missing / departures if departures else 0.0,
        overtime_steps_per_departure=overtime / departures if departures else 0.0,
        declined_per_episode=float(np.mean([r["declined"] for r in records])),
        energy_sold_kwh_per_episode=float(np.mean([r["energy_net_kwh"] for r in records])),
        episodes=episodes,
        config_fingerprint=fingerprint(config, station, dataset),
        per_episode=tuple(records),
    )
