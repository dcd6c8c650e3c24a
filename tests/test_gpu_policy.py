"""The tcgen05 policy kernel (vy_policy_step) against torch references.

* logits / value against a torch restatement of the bf16 autocast forward
  (bf16 operands, fp32 accumulation, bf16 layer outputs) within 2 bf16 ulps
  of the logit scale, and against the plain fp32 network within bf16
  tolerance (3% of the logit scale);
* sampling: each action is the inverse-CDF choice of the documented uniform
  stream over the kernel's own logits (float64 recomputation; only draws
  within 1e-5 of a CDF boundary may differ), log-probabilities within 1e-4;
* the empirical action distribution matches softmax(logits);
* whole, partial (bulk-copy) and ragged (plain-load) tiles; the device call
  counter advances once per launch.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _uniforms(seed, call, n, S):
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed) ^ _mix64(np.uint64(call) + GOLDEN))
        e = np.arange(n * S, dtype=np.uint64)
        x = _mix64(key + e * GOLDEN)
    return (((x >> np.uint64(41)).astype(np.float64) + 0.5) * 2.0 ** -23).astype(np.float32).reshape(n, S)


def _net(scale_head=1.0, seed=0):
    from paper_2507_01522_b200.ppo import ActorCritic

    torch.manual_seed(seed)
    net = ActorCritic(105, 17, 21, 64).cuda()
    with torch.no_grad():
        net.actor[2].weight.mul_(scale_head)
        net.actor[2].bias.normal_(0, 0.05 * scale_head)
        for p in (net.inp.bias, net.actor[0].bias, net.critic[0].bias, net.critic[2].bias):
            p.normal_(0, 0.1)
    return net


def _emulated(net, obs):
    """bf16 autocast forward restated in fp32 on bf16-rounded values."""
    bf = lambda x: x.to(torch.bfloat16).float()  # noqa: E731
    W1 = bf(net.inp.weight)[:, :105]
    h1 = bf(torch.tanh(bf(bf(obs) @ W1.T + bf(net.inp.bias))))
    ha, hc = h1[:, :64], h1[:, 64:]
    h2a = bf(torch.tanh(bf(ha @ bf(net.actor[0].weight).T + bf(net.actor[0].bias))))
    h2c = bf(torch.tanh(bf(hc @ bf(net.critic[0].weight).T + bf(net.critic[0].bias))))
    logits = bf(h2a @ bf(net.actor[2].weight).T[:, :357] + bf(net.actor[2].bias)[:357])
    value = bf(h2c @ bf(net.critic[2].weight)[0] + bf(net.critic[2].bias)[0])
    return logits, value


def _run(net, obs, seed=5, counter=None, logits=True):
    from paper_2507_01522_b200.ppo import pack_policy, policy_step

    N = obs.shape[0]
    counter = counter if counter is not None else torch.zeros(2, dtype=torch.int64, device="cuda")
    a = torch.zeros(N, 17, dtype=torch.uint8, device="cuda")
    lp = torch.zeros(N, device="cuda")
    v = torch.zeros(N, device="cuda")
    lo = torch.full((N, 357), float("nan"), device="cuda") if logits else None
    with torch.no_grad():
        packed = pack_policy(net)
    policy_step(obs, 105, 17, 21, packed, seed, counter, a, lp, v, lo)
    torch.cuda.synchronize()
    return a, lp, v, lo, counter


@pytest.mark.parametrize("N", [4096, 1000, 1001, 77])
def test_policy_forward_matches_bf16_and_fp32_network(N):
    net = _net(scale_head=30.0)
    obs = torch.randn(N, 105, device="cuda") * 2.0
    a, lp, v, lo, ctr = _run(net, obs)
    with torch.no_grad():
        el, ev = _emulated(net, obs)
    scale = float(el.abs().max())
    assert torch.isfinite(lo).all()
    err = (lo - el).abs().max().item()
    assert err <= 2 * 2 ** -8 * scale, (err, scale)
    assert (v - ev).abs().max().item() <= 2 * 2 ** -8 * float(ev.abs().max()) + 1e-3
    with torch.no_grad():  # the plain fp32 network
        fl, fv = net(obs)
    fl = fl.reshape(N, -1)[:, :357]
    assert (lo - fl).abs().max().item() <= 0.03 * scale
    assert (v - fv).abs().max().item() <= 0.03 * float(fv.abs().max()) + 1e-2
    assert int(ctr[0]) == 1 and int(ctr[1]) == 0


@pytest.mark.parametrize("N", [4096, 333])
def test_policy_sampling_is_inverse_cdf_of_the_uniform_stream(N):
    net = _net(scale_head=40.0, seed=1)
    obs = torch.randn(N, 105, device="cuda")
    ctr = torch.tensor([7, 0], dtype=torch.int64, device="cuda")
    a, lp, v, lo, _ = _run(net, obs, seed=123, counter=ctr)
    z = lo.double().cpu().numpy().reshape(N, 17, 21)
    u = _uniforms(123, 7, N, 17).astype(np.float64)
    m = z.max(-1, keepdims=True)
    e = np.exp(z - m)
    ssum = e.sum(-1, keepdims=True)
    cum = np.cumsum(e, -1)
    target = u[..., None] * ssum
    want = np.minimum((cum <= target).sum(-1), 20)
    got = a.cpu().numpy().astype(np.int64)
    bad = got != want
    if bad.any():  # only draws sitting on a CDF boundary (float32 vs float64 sums) may differ
        near = np.abs(cum - target).min(-1) / ssum[..., 0]
        assert (near[bad] < 1e-5).all(), (bad.sum(), near[bad].max())
    assert bad.mean() < 1e-3
    want_lp = (np.take_along_axis(z, got[..., None], -1)[..., 0] - m[..., 0] - np.log(ssum[..., 0])).sum(-1)
    np.testing.assert_allclose(lp.cpu().numpy(), want_lp, rtol=1e-4, atol=1e-4)


def test_policy_action_frequencies_follow_softmax():
    """Identical rows: the empirical action histogram per slot matches softmax(logits)."""
    net = _net(scale_head=20.0, seed=2)
    N = 1 << 15
    obs = torch.randn(1, 105, device="cuda").expand(N, 105).contiguous()
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    a, lp, v, lo, _ = _run(net, obs, counter=ctr)
    z = lo[0].double().cpu().numpy().reshape(17, 21)
    p = np.exp(z - z.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    acts = a.cpu().numpy()
    for s in range(17):
        freq = np.bincount(acts[:, s], minlength=21) / N
        sd = np.sqrt(p[s] * (1 - p[s]) / N)
        assert (np.abs(freq - p[s]) <= 5 * sd + 1e-4).all(), s
    assert torch.equal(v, v[:1].expand(N))


def test_policy_counter_advances_and_streams_differ():
    net = _net(scale_head=30.0, seed=3)
    obs = torch.randn(2048, 105, device="cuda")
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    a0 = _run(net, obs, counter=ctr, logits=False)[0].clone()
    a1 = _run(net, obs, counter=ctr, logits=False)[0].clone()
    assert int(ctr[0]) == 2
    assert (a0 != a1).float().mean() > 0.2  # a new call draws new uniforms


def test_ppo_rollout_fused_policy_env_parity_and_update():
    """PPO with the tcgen05 rollout policy: the env outputs stored by the
    rollout replay bit-exactly on the CPU oracle (the policy only
    chooses the actions), the stored log-probs equal the training forward's
    within bf16 tolerance, and an update runs."""
    from oracle.harness import HostBatch
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PolicyHead, PPOConfig, PPOTrainer

    rc = default_setup(EnvConfig(episode_steps=48), days=30)
    B, T = 512, 64
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=9)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=T, fused_policy=True, use_graph=False))
    ref = HostBatch(env.tables, B, master_seed=9)
    np.testing.assert_array_equal(tr.obs[0].cpu().numpy(), ref.reset().astype(np.float32))
    tr.rollout()
    torch.cuda.synchronize()
    acts = tr.actions.cpu().numpy().astype(np.int64)
    for t in range(T):
        o, r, d = ref.step(acts[t])
        np.testing.assert_array_equal(tr.obs[t + 1].cpu().numpy(), o.astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(tr.rewards[t].cpu().numpy(), r.astype(np.float32))
        np.testing.assert_array_equal(tr.dones[t].cpu().numpy().astype(bool), d)
    # stored log-probs vs the update's (cuBLAS autocast) forward of the same obs / actions
    x = tr.net.pad_obs(tr.obs[:T].reshape(T * B, -1)).to(torch.bfloat16)
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        out, _ = tr.net.forward_merged(x)
        lp, _, v = PolicyHead.apply(out, tr.actions.reshape(T * B, -1), 17, 21, tr.net.out_dim)
    assert (lp - tr.logp.reshape(-1)).abs().max().item() < 0.05
    assert (v - tr.values[:T].reshape(-1)).abs().max().item() < 0.05
    stats = tr.update()
    assert all(torch.isfinite(x).all() for x in stats.values())
    env.close()
