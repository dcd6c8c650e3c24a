"""Energy conservation at scale on the GPU: the reference's acceptance
property (pkg/tests/test_acceptance.py:73-125) over thousands of envs per
station instead of one env per episode, from the device info block.

Per step and occupied port: cap * (soc_after - soc_before) == delivered
(rel 1e-9; a departing car's soc is its departure record); an empty port
delivers exactly 0.  Per env over the episode: the sum of e_net equals the
energy of the departed tenancies plus that of the cars still parked
(rel 1e-6), with tenancies tracked across arrivals and departures."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cases():
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.exogenous import generate_synthetic_defaults
    from paper_2507_01522_b200.station import preset_station
    from paper_2507_01522_b200.workloads import c4_setup

    rc = default_setup(EnvConfig(episode_steps=170), days=30)
    yield "default", rc.env, rc.station, rc.dataset
    yield ("nested_high", EnvConfig(episode_steps=170, allow_discharge=True), preset_station("nested_splitters", 4, 12),
           generate_synthetic_defaults("highway", "high", "eu", seed=1, days=30))
    c4 = c4_setup(days=30)
    yield ("c4_battery", EnvConfig(episode_steps=170, battery_enabled=True, alpha=c4.env.alpha, beta=c4.env.beta),
           c4.station, c4.dataset)


@pytest.mark.parametrize("case", [0, 1, 2])
def test_energy_conservation_at_scale(case):
    from paper_2507_01522_b200 import _native as nat
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    name, cfg, st, ds = list(_cases())[case]
    B = 4096
    env = BatchEnv(cfg, st, ds, batch_size=B, master_seed=11 + case)
    n = env.n_ports
    pol = DeviceRandomPolicy(3 + case, n, cfg.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    env.outs.ensure_info()
    env._bind()
    info = env.outs.info
    S = env.states
    f64 = dict(dtype=torch.float64, device="cuda")

    def caps(meta):
        ids = (meta.long() >> 2)
        lut = torch.tensor([env.profile(p)[0] for p in range(int(ids.max()) + 1)], **f64)
        return lut[ids]

    soc_arr = torch.zeros(n, B, **f64)
    cap_t = torch.zeros(n, B, **f64)
    active = torch.zeros(n, B, dtype=torch.bool, device="cuda")
    departed_delta = torch.zeros(B, **f64)
    e_net_total = torch.zeros(B, **f64)
    rows = torch.arange(B, device="cuda")
    for t in range(cfg.episode_steps - 1):  # the last step would reset the state in the kernel
        meta0 = S.port_meta[:, :B].clone()
        soc0 = S.port_soc[:, :B].clone()
        occ0 = (meta0 & 1).bool()
        cap0 = caps(meta0)
        a = pol.actions(env)
        rc = env._lib.vy_step(env._h, a.data_ptr(), nat.VY_ACT_U8, n + 1, 1, nat.F_AUTO_RESET | nat.F_INFOS, None,
                              env._stream)
        nat.check(rc, "vy_step")
        delivered = info["delivered"][:, :B]
        dep_n = info["dep_n"][:B]
        departed = torch.zeros(n, B, dtype=torch.bool, device="cuda")
        dep_soc = torch.zeros(n, B, **f64)
        for k in range(n):
            ok = k < dep_n
            port = info["dep_port"][k, :B].long().clamp(0, n - 1)
            departed[port[ok], rows[ok]] = True
            dep_soc[port[ok], rows[ok]] = info["dep_soc"][k, :B][ok]
        soc1 = S.port_soc[:, :B]
        soc_after = torch.where(departed, dep_soc, soc1)
        lhs = cap0 * (soc_after - soc0)
        assert torch.all(delivered[~occ0] == 0.0), f"{name}: an empty port delivered energy (t={t})"
        err = (lhs - delivered).abs()
        tol = 1e-9 + 1e-9 * delivered.abs()
        assert bool(torch.all(err[occ0] <= tol[occ0])), f"{name}: per-port energy balance t={t}"
        e_net_total += info["flows"][0, :B]
        # tenancies: close the departed, open the newly occupied
        departed_delta += torch.where(departed & active, cap_t * (dep_soc - soc_arr), 0.0).sum(0)
        active &= ~departed
        occ1 = (S.port_meta[:, :B] & 1).bool()
        new = occ1 & (~occ0 | departed)
        cap1 = caps(S.port_meta[:, :B])
        soc_arr = torch.where(new, soc1, soc_arr)
        cap_t = torch.where(new, cap1, cap_t)
        active |= new
    # tenancies open since reset are complete; cars parked at reset do not exist (reset clears the ports)
    in_station = torch.where(active, cap_t * (S.port_soc[:, :B] - soc_arr), 0.0).sum(0)
    rhs = departed_delta + in_station
    err = (e_net_total - rhs).abs()
    assert bool(torch.all(err <= 1e-9 + 1e-6 * rhs.abs())), f"{name}: episode energy balance"
    env.close()
