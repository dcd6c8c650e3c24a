"""Host-side mirror vs golden vectors produced by the reference.

Pins the table producers the kernels consume: synthetic generators, car
catalogues, scenario models, splitmix64 streams, RandomPolicy draws, and the
flattened step tables (engine.py:107-218) for every golden scenario.
"""

import numpy as np
import pytest

from paper_2507_01522_b200 import exogenous as ex
from paper_2507_01522_b200 import streams
from paper_2507_01522_b200.envconfig import ObsLayout
from paper_2507_01522_b200.streams import BatchStreams, Stream, mix64, split_seed, stream_key
from scenarios import GOLDEN, NAMES, Fixture

SV = np.load(GOLDEN / "synthetic_vectors.npz")


@pytest.mark.parametrize("sc", ex.SCENARIOS)
def test_synthetic_arrivals_and_scenarios(sc):
    for tr in ("low", "medium", "high"):
        a = ex.synthetic_arrivals(sc, tr, dt_min=5)
        np.testing.assert_array_equal(a.rates_per_step, SV[f"arr_{sc}_{tr}"])
        np.testing.assert_array_equal([a.weekday_scale, a.weekend_scale], SV[f"arrscale_{sc}_{tr}"])
    for dtm in (1, 5, 15):
        m = ex.scenario_model(sc, dt_min=dtm)
        got = [*m.stay_steps_range, *m.requested_fraction_range, *m.soc_arrival_range, m.p_charge_sensitive]
        np.testing.assert_array_equal(got, SV[f"scen_{sc}_{dtm}"])


@pytest.mark.parametrize("region", ex.REGIONS)
def test_synthetic_prices_and_catalogue(region):
    for seed in (0, 7):
        p = ex.synthetic_prices(region, seed=seed, days=40)
        np.testing.assert_array_equal(p.buy, SV[f"price_{region}_{seed}"])
        np.testing.assert_array_equal(p.sell_grid, SV[f"sell_{region}_{seed}"])
    np.testing.assert_array_equal(ex.car_catalog(region).cumulative_weights(), SV[f"cum_{region}"])


def test_synthetic_aux():
    a = ex.synthetic_aux(seed=3, days=20)
    np.testing.assert_array_equal(a.moer_kg_per_kwh, SV["aux_moer_3"])
    np.testing.assert_array_equal(a.grid_demand_kwh, SV["aux_dgrid_3"])


def test_stream_known_answers():
    assert mix64(0) == 0
    assert mix64(1) == 0x5692161D100B05E5  # frozen constant, reference tests/test_rng.py:22-26
    assert mix64((1 << 64) - 1) == mix64(-1)
    keys = [stream_key(11, i) for i in range(64)]
    np.testing.assert_array_equal(np.array(keys, dtype=np.uint64), SV["rng_keys"])
    np.testing.assert_array_equal(BatchStreams(np.array(keys, dtype=np.uint64)).uniform_block(9), SV["rng_u"])
    np.testing.assert_array_equal([Stream(k).poisson(3.7) for k in keys], SV["rng_pois"])
    np.testing.assert_array_equal([Stream(k).poisson(70.5) for k in keys], SV["rng_pois_big"])
    got = [split_seed(m, i) for m in (-17, 0, 42) for i in range(8)]
    np.testing.assert_array_equal(np.array(got, dtype=np.uint64), SV["split_seed"])
    assert streams.vstream_key(11, np.arange(64)).tolist() == keys


def test_batch_streams_match_scalar():
    keys = np.array([stream_key(5, i) for i in range(16)], dtype=np.uint64)
    bs = BatchStreams(keys)
    u, ri, po = bs.uniform(), bs.randint(21), bs.poisson(3.0)
    for row, k in enumerate(keys):
        s = Stream(int(k))
        assert u[row] == s.uniform() and ri[row] == s.randint(21) and po[row] == s.poisson(3.0)


def test_poisson_zero_rate_consumes_nothing():
    s = Stream(stream_key(1))
    before = s.state
    assert s.poisson(0.0) == 0 and s.state == before


@pytest.mark.parametrize("name", NAMES)
def test_tables_match_reference_build_tables(name):
    fx = Fixture(name)
    t = fx.tables()
    for key in fx.z.files:
        if not key.startswith("tab_"):
            continue
        field = key[4:]
        want = fx[key]
        got = np.asarray(getattr(t, field))
        np.testing.assert_array_equal(got.astype(want.dtype) if want.dtype != object else got, want,
                                      err_msg=field)
    assert t.obs_len == ObsLayout(t.n_ports, t.horizon).length


def test_fingerprint_matches_reference_reports():
    import json

    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.evaluation import fingerprint

    want = json.loads((GOLDEN / "evaluate_reports.json").read_text())
    rc = default_setup(EnvConfig(episode_steps=96), days=40)
    assert fingerprint(rc.env, rc.station, rc.dataset) == want["idle"]["config_fingerprint"]


@pytest.mark.parametrize("tag", ["default", "c4"])
def test_bridge_observation_space_matches_reference(tag):
    from paper_2507_01522_b200 import DEFAULT_BATTERY, EnvConfig, default_setup, preset_station
    from paper_2507_01522_b200.bridge import MultiDiscreteSpace, observation_space
    from paper_2507_01522_b200.tables import build_tables

    z = np.load(GOLDEN / "bridge_spaces.npz")
    cfg = EnvConfig() if tag == "default" else EnvConfig(battery_enabled=True)
    rc = default_setup(cfg, days=10)
    st = rc.station if tag == "default" else preset_station("nested_splitters", ac_count=0, dc_count=64,
                                                            battery=DEFAULT_BATTERY)
    sp = observation_space(build_tables(cfg, st, rc.dataset))
    np.testing.assert_array_equal(sp.low, z[f"{tag}_low"])
    np.testing.assert_array_equal(sp.high, z[f"{tag}_high"])
    ms = MultiDiscreteSpace(nvec=np.full(17, 21))
    assert ms.contains(np.full(17, 20)) and not ms.contains(np.full(17, 21)) and not ms.contains(np.zeros(17))
