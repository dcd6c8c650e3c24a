"""Device evaluate() and baseline policies vs the reference's evaluate() reports
(tests/golden/evaluate_reports.json, made by scripts/make_golden.py)."""

import json

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from scenarios import GOLDEN  # noqa: E402


@pytest.mark.parametrize("name", ["max_charge", "idle", "random", "max_charge_battery"])
def test_evaluate_matches_reference_report(name):
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.evaluation import evaluate
    from paper_2507_01522_b200.policies import make_policy

    want = json.loads((GOLDEN / "evaluate_reports.json").read_text())[name]
    if name == "max_charge_battery":
        cfg = EnvConfig(episode_steps=48, battery_enabled=True, alpha={"sat0": 1.0}, beta=0.1)
        rc = default_setup(cfg, scenario="highway", traffic="high", days=20)
        rep = evaluate(make_policy("max_charge", 16, 10), rc.env, rc.station, rc.dataset, episodes=40, seed=2)
    else:
        rc = default_setup(EnvConfig(episode_steps=96), days=40)
        rep = evaluate(make_policy(name, 16, 10, seed=3), rc.env, rc.station, rc.dataset, episodes=150, seed=7)
    assert rep.to_dict() == want
