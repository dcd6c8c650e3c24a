"""B200-native vectorised EV charging-station step (Chargax / voltyard hot path).

Host-side mirror of the reference's batched rollout API over hand-written
sm_100a CUDA kernels reached through a C ABI (include/voltyard_b200.h).
"""

from .envconfig import DEFAULT_BATTERY, PENALTY_NAMES, EnvConfig, ObsLayout, RunConfig, default_setup
from .errors import DataError, EpisodeDone, NativeError, SimError, StationError
from .exogenous import (ArrivalProfile, AuxSeries, CarCatalog, CatalogEntry, Dataset, ExogenousFrame,
                        PriceSeries, UserScenarioModel, frame_at, generate_synthetic_defaults,
                        sample_arrival_count, sample_car, sample_user)
from .ingest import (load_arrivals, load_aux, load_car_catalog, load_dataset, load_prices, load_station,
                     save_arrivals, save_aux, save_car_catalog, save_dataset, save_prices, save_station)
from .physics import (BatterySpec, BatteryState, CarProfile, CarState, UserProfile, charge_limit,
                      discharge_limit, integrate_battery, integrate_charge, power_to_current)
from .station import (ArchNode, EvseSpec, StationParams, StationTree, build_station, default_station,
                      enforce_limits, node_load, preset_station, station_from_dict, station_to_dict,
                      violation_excess)
from .streams import BatchStreams, Stream, mix64, split_seed, stream_key
from .tables import StepTables, build_tables

__version__ = "0.1.0"
