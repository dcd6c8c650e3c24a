"""Numerics of the kernels' building blocks on the GPU.

div_rcp replaces IEEE x / d by a precomputed correctly rounded reciprocal
plus one FMA correction; the step's bit-parity depends on it being exactly
the IEEE quotient.  Checked here on 2e8+ random dividends (2^-64..2^64) per
divisor set: every divisor the shipped configs use, plus random divisors.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _divisors_from_configs():
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.tables import build_tables
    from scenarios import NAMES, Fixture

    ds = {1000.0, 365.0}
    tabs = [Fixture(n).tables() for n in NAMES] + [build_tables(*vars(default_setup(EnvConfig(battery_enabled=True))).values())]
    for t in tabs:
        ds.update(t.volt.tolist() + t.eta_c.tolist() + t.i_denom.tolist() + t.node_eta.tolist())
        ds.update(t.cat_cap.tolist() + [1.0 - x for x in t.cat_tau.tolist()])
        ds.update([float(t.episode_steps), t.b_cap, t.b_volt, t.b_eta_c, t.b_idenom, 1.0 - t.b_tau])
    return sorted(d for d in ds if d > 0)


def _run(divs, per, seed):
    from paper_2507_01522_b200 import _native

    arr = (C.c_double * len(divs))(*divs)
    bad = C.c_int64(-1)
    _native.check(_native.lib().vy_selftest_div(arr, len(divs), per, seed, C.byref(bad)), "vy_selftest_div")
    return bad.value


def test_div_rcp_matches_ieee_on_config_divisors():
    divs = _divisors_from_configs()
    assert _run(divs, 4_000_000, 1) == 0


def test_div_rcp_matches_ieee_on_random_divisors():
    rng = np.random.default_rng(0)
    divs = list(np.exp(rng.uniform(np.log(1e-3), np.log(1e6), size=256)))
    divs += [float(x) for x in rng.integers(1, 100000, size=64)]
    assert _run(divs, 1_000_000, 2) == 0
