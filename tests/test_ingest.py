"""Host data ingestion vs files written by the reference (tests/golden/ingest,
made by scripts/make_golden.py::ingest_vectors)."""

import dataclasses
import json

import numpy as np
import pytest

from paper_2507_01522_b200 import DEFAULT_BATTERY, DataError, EnvConfig, preset_station
from paper_2507_01522_b200 import exogenous as ex
from paper_2507_01522_b200 import ingest
from paper_2507_01522_b200.station import station_from_dict, station_to_dict
from paper_2507_01522_b200.tables import build_tables
from scenarios import GOLDEN

ING = GOLDEN / "ingest"


def expected_dataset():
    ds = ex.generate_synthetic_defaults("work", "high", "us", seed=5, days=3)
    return dataclasses.replace(ds, aux=ex.synthetic_aux(seed=1, days=3))


def expected_station():
    st = preset_station("nested_splitters", ac_count=4, dc_count=6, battery=DEFAULT_BATTERY)
    obj = station_to_dict(st)
    obj["evse_order"] = list(reversed([e.id for e in st.evses]))
    return station_from_dict(obj)


def test_load_reference_dataset_dir():
    got, want = ingest.load_dataset(ING / "dataset"), expected_dataset()
    np.testing.assert_array_equal(got.prices.buy, want.prices.buy)
    np.testing.assert_array_equal(got.prices.sell_grid, want.prices.sell_grid)
    assert got.prices.start_date == want.prices.start_date
    np.testing.assert_array_equal(got.arrivals.rates_per_step, want.arrivals.rates_per_step)
    assert (got.arrivals.weekday_scale, got.arrivals.weekend_scale) == (want.arrivals.weekday_scale,
                                                                        want.arrivals.weekend_scale)
    assert got.cars.entries == want.cars.entries
    assert got.scenario == want.scenario
    np.testing.assert_array_equal(got.aux.moer_kg_per_kwh, want.aux.moer_kg_per_kwh)
    np.testing.assert_array_equal(got.aux.grid_demand_kwh, want.aux.grid_demand_kwh)
    cfg = EnvConfig(alpha={"sustain": 0.1, "grid": 0.1})
    st = preset_station("multi_type", 6, 10)
    a, b = build_tables(cfg, st, got), build_tables(cfg, st, want)
    for f in dataclasses.fields(a):
        va, vb = getattr(a, f.name), getattr(b, f.name)
        if isinstance(va, np.ndarray):
            np.testing.assert_array_equal(va, vb, err_msg=f.name)
        else:
            assert va == vb, f.name


def test_save_dataset_is_byte_identical(tmp_path):
    ingest.save_dataset(expected_dataset(), tmp_path)
    for p in sorted((ING / "dataset").iterdir()):
        assert (tmp_path / p.name).read_bytes() == p.read_bytes(), p.name
    back = ingest.load_dataset(tmp_path)
    np.testing.assert_array_equal(back.prices.buy, expected_dataset().prices.buy)


def test_station_json_round_trip(tmp_path):
    st = ingest.load_station(ING / "station.json")
    assert station_to_dict(st) == station_to_dict(expected_station())
    assert st.parking_order == expected_station().parking_order
    ingest.save_station(st, tmp_path / "s.json")
    assert (tmp_path / "s.json").read_bytes() == (ING / "station.json").read_bytes()


@pytest.mark.parametrize("name", sorted(json.loads((ING / "errors.json").read_text())))
def test_loader_errors_match_reference(name, tmp_path):
    case = json.loads((ING / "errors.json").read_text())[name]
    p = tmp_path / case["file"]
    p.write_text(case["text"])
    with pytest.raises(DataError) as ei:
        getattr(ingest, case["loader"])(p)
    assert str(ei.value).replace(str(p), "<path>") == case["error"]


def test_missing_file_is_data_error(tmp_path):
    with pytest.raises(DataError):
        ingest.load_prices(tmp_path / "nope.csv")
