"""The BASELINE.json workloads as (config, station, dataset) triples.

C1/C2/C3 run the default station (``default_setup``: preset multi_type 6 AC +
10 DC, shopping / medium / eu, seed 0, 365 days).
C4 is the large highway station: 64 DC ports under a 3-level splitter tree
(``preset_station("nested_splitters", 0, 64)``, topology.py:323-409) with the
default stationary battery and a profit + satisfaction reward.  C5 is the
heterogeneous sweep in ``hetero.sweep_groups``.
"""

from __future__ import annotations

from .envconfig import DEFAULT_BATTERY, EnvConfig, RunConfig, default_setup
from .exogenous import generate_synthetic_defaults
from .station import preset_station


def c2_setup() -> RunConfig:
    """Default 16-port station (configs C1, C2, C3)."""
    return default_setup()


def c4_setup(days: int = 365) -> RunConfig:
    """64 DC ports, 34-node tree, battery, satisfaction penalties (config C4)."""
    cfg = EnvConfig(battery_enabled=True, alpha={"sat0": 1.0, "sat1": 0.5}, beta=0.2)
    st = preset_station("nested_splitters", ac_count=0, dc_count=64, battery=DEFAULT_BATTERY)
    ds = generate_synthetic_defaults("highway", "high", "eu", seed=0, days=days)
    return RunConfig(env=cfg, station=st, dataset=ds)


__all__ = ["c2_setup", "c4_setup"]
