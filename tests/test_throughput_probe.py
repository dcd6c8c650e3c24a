"""throughput_probe (engine.py:515-556) on the device: the reference's own
tests of the probe (pkg/tests/test_engine.py:156-168; the batch-vs-single
criterion of test_acceptance.py:362-374), its report schema against the
reference's ThroughputReport, and the argument check on CPU."""

import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from scenarios import make_dataset, single_node_station  # noqa: E402


def test_probe_rejects_zero_steps_without_a_device():
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import throughput_probe

    with pytest.raises(ValueError):
        throughput_probe(EnvConfig(), single_node_station(), make_dataset(), total_steps=0)


def test_report_schema_matches_the_reference():
    from paper_2507_01522_b200.batch import ThroughputReport
    from ref_scenarios import import_reference

    ref = import_reference()
    if ref is None:
        pytest.skip("reference not installed in baseline/_ref")
    from voltyard.engine import ThroughputReport as RefReport

    assert [f.name for f in dataclasses.fields(ThroughputReport)] == [f.name for f in dataclasses.fields(RefReport)]
    rep = ThroughputReport(1.0, 2.0, 3, 4, "cuda", 1, "hw")
    assert rep.to_dict() == RefReport(1.0, 2.0, 3, 4, "cuda", 1, "hw").to_dict()


@pytest.mark.gpu
def test_throughput_probe_reports():
    from paper_2507_01522_b200 import EnvConfig
    from paper_2507_01522_b200.batch import throughput_probe

    cfg = EnvConfig(episode_steps=48)
    rep = throughput_probe(cfg, single_node_station(n_ports=3), make_dataset(lam=1.0), batch_size=2,
                           total_steps=500, seed=0)
    assert rep.total_steps >= 500 and rep.total_steps % 2 == 0
    assert rep.steps_per_second > 0 and rep.hardware and rep.backend == "cuda"
    tiny = throughput_probe(cfg, single_node_station(n_ports=3), make_dataset(lam=1.0), batch_size=1,
                            total_steps=1, seed=0)
    assert tiny.total_steps == 1 and np.isfinite(tiny.steps_per_second)


@pytest.mark.gpu
def test_throughput_targets_batch_beats_single():
    """The reference's acceptance criterion (batch-16 >= 1e5 steps/s and >=
    single-env), here with the device batch far above it."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import throughput_probe

    rc = default_setup()
    single = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=1, total_steps=2_000, seed=0)
    batch = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=1 << 16, total_steps=1 << 22, seed=0)
    assert single.wall_seconds <= 10.0
    assert batch.steps_per_second >= 100_000.0
    assert batch.steps_per_second >= single.steps_per_second
