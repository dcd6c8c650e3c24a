"""The fused small-batch PPO update (vy_ppo_update_grad / _adam) against
torch fp32: the flat gradient of one minibatch equals torch autograd of the
same clipped PPO loss (log-softmax per slot, entropy bonus, advantages
normalised over the minibatch, clipped value loss) within fp32 tolerance —
on a fresh network and on one with large logits (saturated tanh, clipped
ratios); the Adam step (clip_grad_norm_ + Adam, bias-corrected) equals
torch.optim.Adam given the same gradient; and the trainer with the fused
update learns and replays its update graph."""

import ctypes as C

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _data(n, obs_dim, S, A, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    obs = torch.rand(n, obs_dim, device="cuda", generator=g) * 2 - 1
    act = torch.randint(0, A, (n, S), device="cuda", generator=g, dtype=torch.uint8)
    scal = torch.randn(n, 4, device="cuda", generator=g)
    scal[:, 0] = scal[:, 0] * 3 - 40  # old log-probabilities around the uniform policy's 17 * log(1/21)
    return obs, act, scal.contiguous()


def _torch_loss(net, obs, act, scal, idx, cfg):
    from paper_2507_01522_b200.ppo import head_reference

    logits, v = net(obs[idx], logits_fp32=True)
    lp, ent = head_reference(logits, act[idx])
    old_lp, old_v, a, r = scal[idx].unbind(1)
    a = (a - a.mean()) / (a.std() + 1e-8)
    ratio = torch.exp(lp - old_lp)
    pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip_eps, 1 + cfg.clip_eps) * a).mean()
    v_clip = old_v + (v - old_v).clamp(-cfg.vf_clip, cfg.vf_clip)
    vl = 0.5 * torch.max((v - r) ** 2, (v_clip - r) ** 2).mean()
    ent = ent.mean()
    return pg + cfg.vf_coef * vl - cfg.ent_coef * ent, (pg, vl, ent)


def _fused_grad(net, obs, act, scal, idx, cfg, step):
    from paper_2507_01522_b200 import _native as nat

    S, A, od = net.n_slots, net.n_actions, net.obs_dim
    M = idx.numel()
    ws = (C.c_int64 * 4)()
    assert nat.lib().vy_ppo_update_workspace(od, S, A, 64, M, ws) == nat.VY_OK
    work = torch.zeros(ws[1], device="cuda")
    grad = torch.zeros(ws[0], device="cuda")
    stats = torch.zeros(4, device="cuda")
    prm = list(net.parameters())
    ptrs = (C.c_void_p * len(prm))(*[p.data_ptr() for p in prm])
    w1t = net.inp.weight.detach().t().contiguous()
    nat.check(nat.lib().vy_ppo_update_grad(ptrs, w1t.data_ptr(), od, S, A, 64, obs.data_ptr(), obs.stride(0), act.data_ptr(),
                                           scal.data_ptr(), idx.data_ptr(), None, M, cfg.clip_eps, cfg.vf_clip,
                                           cfg.vf_coef, cfg.ent_coef, work.data_ptr(), grad.data_ptr(),
                                           stats.data_ptr(), step.data_ptr(), torch.cuda.current_stream().cuda_stream),
              "vy_ppo_update_grad")
    return grad, stats, work, w1t


@pytest.mark.parametrize("M,scale", [(1200, 1.0), (75, 1.0), (900, 30.0), (37, 1.0), (2000, 1.0)])
def test_fused_gradient_matches_torch_fp32(M, scale):
    from paper_2507_01522_b200.ppo import ActorCritic, PPOConfig

    torch.manual_seed(3)
    S, A, od = 17, 21, 105
    net = ActorCritic(od, S, A).cuda()
    if scale != 1.0:  # large logits and pre-activations: saturated tanh, far-from-1 ratios (clipped branches)
        with torch.no_grad():
            net.actor[2].weight.mul_(scale)
            net.inp.weight.mul_(3.0)
    cfg = PPOConfig()
    obs, act, scal = _data(4 * M, od, S, A, seed=M)
    idx = torch.randperm(4 * M, device="cuda")[:M].contiguous()
    step = torch.zeros(1, device="cuda")
    grad, stats, _, _ = _fused_grad(net, obs, act, scal, idx, cfg, step)
    loss, (pg, vl, ent) = _torch_loss(net, obs, act, scal, idx, cfg)
    net.zero_grad()
    loss.backward()
    ref = torch.cat([p.grad.reshape(-1) for p in net.parameters()])
    assert torch.isfinite(grad).all()
    err = (grad - ref).abs().max().item()
    tol = 2e-4 * ref.abs().max().item() + 1e-6
    assert err <= tol, f"max |grad - torch| = {err:.3e} (tol {tol:.3e})"
    cos = torch.nn.functional.cosine_similarity(grad, ref, dim=0).item()
    assert cos > 0.99999, cos
    torch.testing.assert_close(stats, torch.stack([loss, pg, vl, ent]).detach(), rtol=2e-4, atol=2e-5)
    assert step.item() == 1.0


def test_fused_adam_matches_torch_adam():
    from paper_2507_01522_b200 import _native as nat
    from paper_2507_01522_b200.ppo import ActorCritic, PPOConfig

    torch.manual_seed(5)
    S, A, od, M = 17, 21, 105, 600
    net = ActorCritic(od, S, A).cuda()
    ref = ActorCritic(od, S, A).cuda()
    ref.load_state_dict(net.state_dict())
    cfg = PPOConfig(max_grad_norm=0.05)  # small: the clip coefficient is active
    lr = torch.tensor(3e-4, device="cuda")
    opt = torch.optim.Adam(ref.parameters(), lr=3e-4, eps=1e-5)
    m = torch.zeros(sum(p.numel() for p in net.parameters()), device="cuda")
    v = torch.zeros_like(m)
    step = torch.zeros(1, device="cuda")
    obs, act, scal = _data(4 * M, od, S, A, seed=11)
    for it in range(3):
        idx = torch.randperm(4 * M, device="cuda")[:M].contiguous()
        grad, _, work, w1t = _fused_grad(net, obs, act, scal, idx, cfg, step)
        # the reference optimiser gets exactly the fused gradient
        off = 0
        for p in ref.parameters():
            p.grad = grad[off:off + p.numel()].view_as(p).clone()
            off += p.numel()
        torch.nn.utils.clip_grad_norm_(ref.parameters(), cfg.max_grad_norm)
        opt.step()
        prm = list(net.parameters())
        pp = (C.c_void_p * len(prm))(*[p.data_ptr() for p in prm])
        nat.check(nat.lib().vy_ppo_update_adam(pp, w1t.data_ptr(), od, S, A, 64, M, work.data_ptr(), grad.data_ptr(), m.data_ptr(),
                                               v.data_ptr(), lr.data_ptr(), step.data_ptr(), 0.9, 0.999, 1e-5,
                                               cfg.max_grad_norm, torch.cuda.current_stream().cuda_stream),
                  "vy_ppo_update_adam")
        for (name, a), b in zip(net.named_parameters(), ref.parameters()):
            torch.testing.assert_close(a, b, rtol=1e-5, atol=2e-7, msg=f"{name} after step {it + 1}")
        assert torch.equal(w1t, net.inp.weight.detach().t())  # the transposed copy follows the update exactly
    assert step.item() == 3.0


def test_trainer_fused_update_learns_and_replays():
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup()
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=16, master_seed=0)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=300, total_timesteps=40 * 300 * 16))
    assert tr._fused_update and "vy_ppo_update_grad" in tr.describe_update()
    w0 = [p.detach().clone() for p in tr.net.parameters()]
    ents = []
    for _ in range(8):
        st = tr.iterate()
        assert all(torch.isfinite(v).all() for v in st.values())
        ents.append(float(st["ent"]))
    moved = sum((p - q).abs().sum().item() for p, q in zip(tr.net.parameters(), w0))
    assert moved > 0
    assert ents[-1] < ents[0]  # the policy sharpens from the near-uniform start
    assert tr._adam_step.item() == 8 * 4 * 4  # iterations x epochs x minibatches optimizer steps
    env.close()


def test_trainer_fused_update_equals_eager_replay():
    """The captured update graph and the eager fused update give the same
    weights from the same rollout data (same permutation stream)."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup()
    trs = []
    for graph in (False, True):
        env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=16, master_seed=2)
        trs.append(PPOTrainer(env, PPOConfig(rollout_steps=100, use_graph=graph, graph_update=graph)))
    assert trs[1]._graph_update and not trs[0]._graph_update
    trs[0].rollout()
    for name in ("obs", "actions", "logp", "values", "rewards", "dones"):  # the same rollout data in both
        getattr(trs[1], name).copy_(getattr(trs[0], name))
    for tr in trs:  # identical networks (seeded init), the same permutation stream
        torch.manual_seed(7)
        tr.update()  # graph trainer: the eager warm-up update, then the capture (not executed)
    for a, b in zip(trs[0].net.parameters(), trs[1].net.parameters()):
        assert torch.equal(a, b)
    for tr in trs:
        tr.env.close()


@pytest.mark.parametrize("n", [1, 2, 300, 4800, 16384, 100003])
def test_random_perms_are_permutations(n):
    from paper_2507_01522_b200 import _native as nat

    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = torch.empty(4, n, dtype=torch.int64, device="cuda")
    seen = []
    for _ in range(2):
        nat.check(nat.lib().vy_random_perms(n, 4, 123, ctr.data_ptr(), out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream), "vy_random_perms")
        for row in out:
            assert torch.equal(torch.sort(row).values, torch.arange(n, device="cuda"))
        seen.append(out.clone())
    assert ctr.tolist() == [2, 0]
    if n >= 300:
        rows = torch.cat(seen)
        assert len({tuple(r[:16].tolist()) for r in rows}) == 8  # every draw differs
        # shuffled, not structured: each draw is uncorrelated with the identity
        # (|r| ~ 1/sqrt(n)) and has few fixed points (~1 expected)
        ar = torch.arange(n, device="cuda", dtype=torch.float64)
        for r in rows.double():
            corr = torch.corrcoef(torch.stack([ar, r]))[0, 1].item()
            assert abs(corr) < 4.0 / n ** 0.5, corr
            assert (r == ar).sum().item() < 10


def test_precomputed_advantage_stats_match_in_kernel():
    """vy_ppo_adv_stats (every minibatch of an update at once) gives the
    minibatch mean / unbiased std torch computes, and the gradient computed
    with them equals the in-kernel statistics' to fp32 rounding."""
    from paper_2507_01522_b200 import _native as nat
    from paper_2507_01522_b200.ppo import ActorCritic, PPOConfig

    torch.manual_seed(9)
    S, A, od, n, E, nmb = 17, 21, 105, 4800, 2, 4
    mb = n // nmb
    obs, act, scal = _data(n, od, S, A, seed=21)
    perms = torch.stack([torch.randperm(n, device="cuda") for _ in range(E)]).contiguous()
    out = torch.zeros(E * nmb, 2, device="cuda")
    nat.check(nat.lib().vy_ppo_adv_stats(scal.data_ptr(), perms.data_ptr(), n, E, nmb, mb, out.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream), "vy_ppo_adv_stats")
    for e in range(E):
        for k in range(nmb):
            a = scal[perms[e, k * mb:(k + 1) * mb], 2]
            torch.testing.assert_close(out[e * nmb + k], torch.stack([a.mean(), a.std()]), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("T,B", [(300, 16), (300, 1), (64, 4096)])
def test_gae_scal_equals_gae(T, B):
    """vy_gae_scal (the fused update's GAE, one block for small rollouts)
    writes {logp, value, advantage, return} rows bit-identical to vy_gae."""
    from paper_2507_01522_b200 import _native as nat
    from paper_2507_01522_b200.ppo import gae

    g = torch.Generator(device="cuda").manual_seed(B)
    values = torch.randn(T + 1, B, device="cuda", generator=g)
    rewards = torch.randn(T, B, device="cuda", generator=g)
    dones = (torch.rand(T, B, device="cuda", generator=g) < 0.05).to(torch.uint8)
    logp = torch.randn(T, B, device="cuda", generator=g)
    adv, ret = gae(values[:T], rewards, dones, values[T], 0.99, 0.95)
    scal = torch.empty(T * B, 4, device="cuda")
    nat.check(nat.lib().vy_gae_scal(values.data_ptr(), rewards.data_ptr(), dones.data_ptr(), values[T].data_ptr(),
                                    logp.data_ptr(), T, B, 0.99, 0.95, scal.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "vy_gae_scal")
    want = torch.stack([logp.reshape(-1), values[:T].reshape(-1), adv.reshape(-1), ret.reshape(-1)], 1)
    assert torch.equal(scal, want)
