"""PPO support on the GPU (config C3): GAE kernel, graph-captured rollouts.

The rollout test replays the actions the policy sampled inside the captured
CUDA graph on the CPU oracle and requires the env outputs stored in the
rollout buffers to equal float32(oracle) exactly — the graph path is the same
bit-exact env step.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_gae_kernel_matches_torch_restatement():
    from paper_2507_01522_b200.ppo import gae, gae_reference

    g = torch.Generator(device="cuda").manual_seed(0)
    T, B = 37, 1000
    v = torch.randn(T, B, device="cuda", generator=g)
    r = torch.randn(T, B, device="cuda", generator=g)
    d = (torch.rand(T, B, device="cuda", generator=g) < 0.05).to(torch.uint8)
    lv = torch.randn(B, device="cuda", generator=g)
    a1, r1 = gae(v, r, d, lv, 0.99, 0.95)
    a2, r2 = gae_reference(v, r, d, lv, 0.99, 0.95)
    torch.testing.assert_close(a1, a2, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(r1, r2, rtol=1e-5, atol=1e-5)


def test_eager_rollout_buffers_replay_on_oracle():
    from oracle.harness import HostBatch
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup(EnvConfig(episode_steps=24), days=30)
    B, T = 64, 40
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=4)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=T, use_graph=False, total_timesteps=10 * T * B))
    ref = HostBatch(env.tables, B, master_seed=4)
    ref.reset()
    np.testing.assert_array_equal(tr.obs[0].cpu().numpy(), ref.outs.obs.astype(np.float32))
    tr.rollout()
    acts = tr.actions.cpu().numpy().astype(np.int64)
    obs, rew, done = tr.obs.cpu().numpy(), tr.rewards.cpu().numpy(), tr.dones.cpu().numpy()
    for t in range(T):
        o, r, d = ref.step(acts[t])
        np.testing.assert_array_equal(obs[t + 1], o.astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(rew[t], r.astype(np.float32))
        np.testing.assert_array_equal(done[t], d.astype(np.uint8))
    assert np.isfinite(tr.values.cpu().numpy()).all()
    stats = tr.update()
    assert all(torch.isfinite(v) for v in stats.values())
    env.close()


def test_graph_rollout_continues_env_exactly():
    """Two graph replays = 2T env steps: replay every recorded action on the oracle
    from a state snapshot taken before the second replay."""
    from oracle.harness import HostBatch
    from paper_2507_01522_b200 import EnvConfig, default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup(EnvConfig(episode_steps=24), days=30)
    B, T = 64, 30
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=8)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=T, use_graph=True, total_timesteps=10 * T * B))
    tr.rollout()  # warm-up + capture + first replay
    # the host lockstep clock follows the GPU's step counter (warm-up included)
    assert env._t == int(env.states.view("step")[0])
    tr.obs[0].copy_(tr.obs[T])
    before = env.reference_state()
    tr.rollout()  # second replay
    assert env._t == int(env.states.view("step")[0])
    acts = tr.actions.cpu().numpy().astype(np.int64)
    # CPU oracle started from the device state snapshot
    ref = HostBatch(env.tables, B, master_seed=8)
    for k, v in before.items():
        getattr(ref.states, k)[...] = v
    ref._needs_reset = False
    obs, rew = tr.obs.cpu().numpy(), tr.rewards.cpu().numpy()
    for t in range(T):
        o, r, d = ref.step(acts[t])
        np.testing.assert_array_equal(obs[t + 1], o.astype(np.float32), err_msg=f"t={t}")
        np.testing.assert_array_equal(rew[t], r.astype(np.float32))
    env.close()


def test_ppo_learns_a_little():
    """A few iterations move the policy (loss finite, entropy decreasing from uniform)."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup()
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=1024, master_seed=0)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=64, total_timesteps=20 * 64 * 1024))
    ents = [float(tr.iterate()["ent"]) for _ in range(6)]
    assert all(np.isfinite(ents))
    assert ents[-1] < ents[0]
    env.close()


def test_fused_policy_head_matches_torch_fp32():
    """vy_ppo_head_fwd/_bwd against the plain torch fp32 log-softmax head:
    log-probabilities, entropies and the logits gradient of a mixed loss."""
    from paper_2507_01522_b200.ppo import PolicyHead, head_reference

    g = torch.Generator(device="cuda").manual_seed(0)
    N, S, A = 5000, 17, 21
    z = (torch.randn(N, S, A, device="cuda", generator=g) * 3).requires_grad_(True)
    a = torch.randint(0, A, (N, S), device="cuda", generator=g).to(torch.uint8)
    w1, w2 = torch.randn(N, device="cuda", generator=g), torch.randn(N, device="cuda", generator=g)
    lp, ent = PolicyHead.apply(z, a, S, A)
    (lp * w1 + ent * w2).sum().backward()
    gz = z.grad.clone()
    z.grad = None
    lp_r, ent_r = head_reference(z, a)
    (lp_r * w1 + ent_r * w2).sum().backward()
    torch.testing.assert_close(lp, lp_r, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(ent, ent_r, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(gz, z.grad, rtol=1e-4, atol=1e-5)


def test_fused_sampler_is_gumbel_max():
    """vy_ppo_sample picks argmax(logits + Gumbel(noise)) per slot and returns
    the summed log-softmax of the picks (torch fp32 reference)."""
    from paper_2507_01522_b200 import _native as nat

    g = torch.Generator(device="cuda").manual_seed(1)
    N, S, A = 4096, 17, 21
    z = torch.randn(N, S, A, device="cuda", generator=g) * 2
    u = torch.rand(N, S, A, device="cuda", generator=g)
    act = torch.empty(N, S, dtype=torch.uint8, device="cuda")
    lp = torch.empty(N, device="cuda")
    nat.check(nat.lib().vy_ppo_sample(z.data_ptr(), 0, S * A, u.data_ptr(), N, S, A, act.data_ptr(), lp.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "vy_ppo_sample")
    ref = torch.argmax(z - torch.log(-torch.log(u.clamp(1e-20, 1.0))), dim=-1)
    assert (act.long() == ref).float().mean() > 0.9999  # fast-math log may flip exact near-ties only
    lp_r = torch.log_softmax(z, -1).gather(-1, act.long().unsqueeze(-1)).squeeze(-1).sum(-1)
    torch.testing.assert_close(lp, lp_r, rtol=1e-5, atol=1e-4)


def test_fused_policy_head_bf16_logits():
    """bf16 logits (the autocast GEMM output) go straight into the head: the
    result equals the fp32 head on the upcast logits; the gradient comes back
    in bf16 (what autograd's cast would have produced from the fp32 one)."""
    from paper_2507_01522_b200.ppo import PolicyHead

    g = torch.Generator(device="cuda").manual_seed(2)
    N, S, A = 3000, 17, 21
    zb = (torch.randn(N, S, A, device="cuda", generator=g) * 3).to(torch.bfloat16).requires_grad_(True)
    zf = zb.detach().float().requires_grad_(True)
    a = torch.randint(0, A, (N, S), device="cuda", generator=g).to(torch.uint8)
    w1, w2 = torch.randn(N, device="cuda", generator=g), torch.randn(N, device="cuda", generator=g)
    lpb, entb = PolicyHead.apply(zb, a, S, A)
    (lpb * w1 + entb * w2).sum().backward()
    lpf, entf = PolicyHead.apply(zf, a, S, A)
    (lpf * w1 + entf * w2).sum().backward()
    torch.testing.assert_close(lpb, lpf, rtol=0, atol=0)
    torch.testing.assert_close(entb, entf, rtol=0, atol=0)
    assert zb.grad.dtype == torch.bfloat16
    torch.testing.assert_close(zb.grad, zf.grad.to(torch.bfloat16), rtol=0, atol=0)


def test_fused_policy_head_padded_rows():
    """Logits read in place from a GEMM output padded to an aligned width: the
    same values as the packed rows, zero gradient in the padding columns."""
    from paper_2507_01522_b200.ppo import PolicyHead

    g = torch.Generator(device="cuda").manual_seed(3)
    N, S, A, W = 2000, 17, 21, 360
    full = (torch.randn(N, W, device="cuda", generator=g)).to(torch.bfloat16).requires_grad_(True)
    packed = full.detach()[:, : S * A].contiguous().requires_grad_(True)
    a = torch.randint(0, A, (N, S), device="cuda", generator=g).to(torch.uint8)
    w1 = torch.randn(N, device="cuda", generator=g)
    lp1, e1 = PolicyHead.apply(full, a, S, A)
    (lp1 * w1 + e1).sum().backward()
    lp2, e2 = PolicyHead.apply(packed, a, S, A)
    (lp2 * w1 + e2).sum().backward()
    torch.testing.assert_close(lp1, lp2, rtol=0, atol=0)
    torch.testing.assert_close(full.grad[:, : S * A], packed.grad, rtol=0, atol=0)
    assert (full.grad[:, S * A:] == 0).all()


@pytest.mark.parametrize("autocast", [False, True])
def test_linear_gemm_bias_grad_matches_torch(autocast):
    """The update's linear layers (bias gradient as a ones-row GEMM) give torch's
    gradients: fp32 tightly, bf16 autocast within bf16 rounding."""
    from paper_2507_01522_b200.ppo import _Linear

    torch.manual_seed(0)
    lin = _Linear(112, 360).cuda()
    ref = torch.nn.Linear(112, 360).cuda()
    ref.load_state_dict(lin.state_dict())
    x = torch.randn(4099, 112, device="cuda", requires_grad=True)
    x2 = x.detach().clone().requires_grad_(True)
    g = torch.randn(4099, 360, device="cuda")
    with torch.autocast("cuda", dtype=torch.bfloat16, enabled=autocast):
        y = lin(x)
        y2 = ref(x2)
    (y.float() * g).sum().backward()
    (y2.float() * g).sum().backward()
    tol = dict(rtol=2e-2, atol=2e-2) if autocast else dict(rtol=1e-4, atol=1e-3)
    torch.testing.assert_close(y.float(), y2.float(), **tol)
    scale = lambda t: t / t.abs().max()  # noqa: E731
    torch.testing.assert_close(scale(lin.weight.grad), scale(ref.weight.grad), **tol)
    torch.testing.assert_close(scale(lin.bias.grad), scale(ref.bias.grad), **tol)
    torch.testing.assert_close(scale(x.grad), scale(x2.grad), **tol)


def test_gather_rows_equals_indexing():
    from paper_2507_01522_b200.ppo import gather_rows

    src = torch.randn(5000, 112, device="cuda").to(torch.bfloat16)
    idx = torch.randint(0, 5000, (3001,), device="cuda")
    torch.testing.assert_close(gather_rows(src, idx), src[idx], rtol=0, atol=0)
    assert gather_rows(src, idx[:0]).shape == (0, 112)
    with pytest.raises(ValueError):
        gather_rows(src[:, :7], idx)


def test_in_kernel_rng_sampler_draws_the_softmax():
    """vy_ppo_sample_rng: action frequencies follow softmax(logits), the
    log-probability is that of the pick, the device call counter advances once
    per launch, and (seed, call) reproduces the draw."""
    from paper_2507_01522_b200 import _native as nat

    N, S, A = 1 << 16, 3, 5
    z = torch.tensor([0.0, 1.0, -1.0, 2.0, 0.5], device="cuda").repeat(N, S, 1).contiguous()
    probs = torch.softmax(z[0, 0], -1)
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def draw():
        act = torch.empty(N, S, dtype=torch.uint8, device="cuda")
        lp = torch.empty(N, device="cuda")
        nat.check(nat.lib().vy_ppo_sample_rng(z.data_ptr(), 0, S * A, 1234, ctr.data_ptr(), N, S, A,
                                              act.data_ptr(), lp.data_ptr(), None, 0, st), "vy_ppo_sample_rng")
        return act, lp

    a1, lp1 = draw()
    assert ctr.tolist() == [1, 0]
    a2, _ = draw()
    assert ctr.tolist() == [2, 0]
    assert (a1 != a2).float().mean() > 0.3
    freq = torch.bincount(a1.long().reshape(-1), minlength=A).float() / (N * S)
    torch.testing.assert_close(freq, probs, rtol=0, atol=6e-3)  # ~5 sigma at 196k draws
    lp_r = torch.log_softmax(z, -1).gather(-1, a1.long().unsqueeze(-1)).squeeze(-1).sum(-1)
    torch.testing.assert_close(lp1, lp_r, rtol=1e-5, atol=1e-4)
    ctr.zero_()
    a3, _ = draw()
    assert torch.equal(a1, a3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_colsum_matches_torch(dtype):
    from paper_2507_01522_b200.ppo import colsum

    g = torch.randn(30001, 360, device="cuda").to(dtype)
    torch.testing.assert_close(colsum(g), g.float().sum(0), rtol=1e-4, atol=1e-2)
    torch.testing.assert_close(colsum(g[:, :357]), g[:, :357].float().sum(0), rtol=1e-4, atol=1e-2)
    torch.testing.assert_close(colsum(g[:5, :1]), g[:5, :1].float().sum(0), rtol=1e-4, atol=1e-4)
    assert torch.equal(colsum(g), colsum(g))  # no atomics: bit-identical run to run
    assert torch.equal(colsum(g[:0]), torch.zeros(360, device="cuda"))


def test_rollout_inference_weights_match_the_network():
    """The rollout's three-GEMM forward (block-diagonal second layer, merged
    heads) gives the network's logits and value to bf16 accuracy."""
    from paper_2507_01522_b200.ppo import ActorCritic

    torch.manual_seed(0)
    net = ActorCritic(105, 17, 21).cuda()
    for p in net.parameters():  # non-trivial biases and head weights
        p.data.add_(0.05 * torch.randn_like(p))
    x = torch.zeros(512, net.in_dim, device="cuda")
    x[:, :105] = torch.randn(512, 105, device="cuda")
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits, v = net(x, logits_fp32=False)
        out, v2 = net.infer(x.to(torch.bfloat16), net.inference_weights())
    assert out.shape == (512, net.out_dim + 8) and out.stride(0) == net.out_dim + 8
    torch.testing.assert_close(out[:, : net.n_out].float(), logits[:, : net.n_out].float(), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(v2.float(), v.float(), rtol=2e-2, atol=2e-2)


def test_merged_training_forward_matches_the_network():
    """forward_merged (block-diagonal layer 2, merged heads) gives the same
    outputs and parameter gradients as the layer-by-layer forward (fp32)."""
    from paper_2507_01522_b200.ppo import ActorCritic

    torch.manual_seed(1)
    net = ActorCritic(105, 17, 21).cuda()
    for p in net.parameters():
        p.data.add_(0.05 * torch.randn_like(p))
    x = torch.zeros(777, net.in_dim, device="cuda")
    x[:, :105] = torch.randn(777, 105, device="cuda")
    gl = torch.randn(777, net.n_out, device="cuda")
    gv = torch.randn(777, device="cuda")
    logits, v = net(x, logits_fp32=False)
    ((logits[:, : net.n_out] * gl).sum() + (v * gv).sum()).backward()
    ref = {n: p.grad.clone() for n, p in net.named_parameters()}
    net.zero_grad()
    out, v2 = net.forward_merged(x)
    ((out[:, : net.n_out] * gl).sum() + (v2 * gv).sum()).backward()
    torch.testing.assert_close(out[:, : net.n_out], logits[:, : net.n_out], rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(v2, v, rtol=1e-4, atol=1e-4)
    for n, p in net.named_parameters():
        torch.testing.assert_close(p.grad, ref[n], rtol=1e-3, atol=1e-3, msg=n)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_policy_head_value_column(dtype):
    """PolicyHead with value_col: the value is column value_col of the rows and
    its gradient lands there in the same backward pass; the logits gradient
    equals the plain head plus a column select."""
    from paper_2507_01522_b200.ppo import PolicyHead

    torch.manual_seed(2)
    N, S, A, ld, col = 3001, 17, 21, 368, 360
    base = torch.randn(N, ld, device="cuda").to(dtype)
    a = torch.randint(0, A, (N, S), device="cuda", dtype=torch.uint8)
    g1, g2, g3 = (torch.randn(N, device="cuda") for _ in range(3))
    z1 = base.clone().requires_grad_(True)
    lp, ent, v = PolicyHead.apply(z1, a, S, A, col)
    ((lp * g1).sum() + (ent * g2).sum() + (v * g3).sum()).backward()
    z2 = base.clone().requires_grad_(True)
    lp2, ent2 = PolicyHead.apply(z2, a, S, A)
    v2 = z2[:, col].float()
    ((lp2 * g1).sum() + (ent2 * g2).sum() + (v2 * g3).sum()).backward()
    torch.testing.assert_close(v, v2, rtol=0, atol=0)
    torch.testing.assert_close(lp, lp2, rtol=0, atol=0)
    torch.testing.assert_close(z1.grad.float(), z2.grad.float(), rtol=1e-2, atol=1e-2)
    assert torch.equal(z1.grad[:, col].float(), g3.to(dtype).float())


def test_sampler_writes_the_value_column():
    from paper_2507_01522_b200 import _native as nat

    N, S, A, ld, col = 1000, 17, 21, 368, 360
    z = torch.randn(N, ld, device="cuda").to(torch.bfloat16)
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    act = torch.empty(N, S, dtype=torch.uint8, device="cuda")
    lp = torch.empty(N, device="cuda")
    val = torch.empty(N, device="cuda")
    nat.check(nat.lib().vy_ppo_sample_rng(z.data_ptr(), 1, ld, 7, ctr.data_ptr(), N, S, A, act.data_ptr(),
                                          lp.data_ptr(), val.data_ptr(), col,
                                          torch.cuda.current_stream().cuda_stream), "vy_ppo_sample_rng")
    assert torch.equal(val, z[:, col].float())


@pytest.mark.parametrize("fused,graph", [(False, True), (False, False), (True, False)])
def test_trainer_non_default_modes_run(fused, graph):
    """The torch-head and eager (no CUDA graph) trainer paths still run and
    give finite losses."""
    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    rc = default_setup()
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=256, master_seed=1)
    tr = PPOTrainer(env, PPOConfig(rollout_steps=20, fused_head=fused, fused_policy=fused, use_graph=graph))
    for _ in range(2):
        st = tr.iterate()
    assert all(torch.isfinite(v).all() for v in st.values())
    env.close()


def test_update_graph_with_captured_nccl_allreduce():
    """The multi-GPU update path on one GPU: a 1-rank NCCL group with the
    per-minibatch gradient all-reduce forced on, captured inside the update
    CUDA graph.  SUM / 1 is exact, so the weights after two iterations equal
    the all-reduce-free trainer's bit for bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv
    from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rc = default_setup()
        weights = []
        for mode in ("always", "auto"):
            env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=512, master_seed=2)
            tr = PPOTrainer(env, PPOConfig(rollout_steps=32, allreduce=mode))
            assert tr._graph_update and tr._allreduce == (mode == "always")
            for _ in range(3):
                st = tr.iterate()
            assert all(torch.isfinite(v).all() for v in st.values())
            weights.append([p.detach().clone() for p in tr.net.parameters()])
            env.close()
        for a, b in zip(*weights):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,A,N", [(17, 21, 3001), (9, 21, 2500), (17, 7, 700)])
def test_fused_ppo_loss_matches_torch(S, A, N):
    """vy_ppo_loss (PPOLoss): the minibatch loss, its parts and d loss / d head
    rows equal the torch restatement (log-softmax head, clipped surrogate,
    clipped value loss, entropy bonus; advantages normalised per minibatch)
    within bf16 / fast-math tolerances, ratios on both sides of the clip."""
    from paper_2507_01522_b200.ppo import PPOLoss, head_reference

    torch.manual_seed(3)
    vcol, ld = S * A, S * A + 11  # value in a padding column, padded row stride
    dev = "cuda"
    raw = (torch.randn(N, ld, device=dev) * 1.5).to(torch.bfloat16)
    act = torch.randint(0, A, (N, S), device=dev, dtype=torch.uint8)
    with torch.no_grad():
        lp0, _ = head_reference(raw[:, :S * A].float().view(N, S, A), act)
    old_lp = lp0 + 0.3 * torch.randn(N, device=dev)  # ratios around 1, many beyond 1 +- 0.2
    old_v = raw[:, vcol].float() + 4.0 * torch.randn(N, device=dev)  # some value updates clipped at 10
    adv = torch.randn(N, device=dev) * 2 + 0.3
    ret = torch.randn(N, device=dev) * 5
    scal = torch.stack([old_lp, old_v, adv, ret], 1).contiguous()
    adv_stats = torch.stack([adv.mean(), adv.std()])
    cfg = dict(clip_eps=0.2, vf_clip=10.0, vf_coef=0.25, ent_coef=0.01)

    logits = raw.clone().requires_grad_()
    loss, means = PPOLoss.apply(logits, act, scal, adv_stats, S, A, vcol, cfg["clip_eps"], cfg["vf_clip"],
                                cfg["vf_coef"], cfg["ent_coef"])
    (3.0 * loss).backward()  # a non-unit upstream gradient scales the stored one

    lg = raw.float().requires_grad_()
    lp, ent = head_reference(lg[:, :S * A].reshape(N, S, A), act)
    v = lg[:, vcol]
    a = (adv - adv.mean()) / (adv.std() + 1e-8)
    ratio = torch.exp(lp - old_lp)
    pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg["clip_eps"], 1 + cfg["clip_eps"]) * a).mean()
    v_clip = old_v + (v - old_v).clamp(-cfg["vf_clip"], cfg["vf_clip"])
    vl = 0.5 * torch.max((v - ret) ** 2, (v_clip - ret) ** 2).mean()
    ent_m = ent.mean()
    ref = pg + cfg["vf_coef"] * vl - cfg["ent_coef"] * ent_m
    (3.0 * ref).backward()

    torch.testing.assert_close(loss, ref.detach(), rtol=2e-4, atol=1e-5)
    torch.testing.assert_close(means, torch.stack([pg, vl, ent_m]).detach(), rtol=2e-4, atol=1e-5)
    g = logits.grad.float()
    want = lg.grad.to(torch.bfloat16).float()
    torch.testing.assert_close(g[:, :S * A], want[:, :S * A], rtol=2e-2, atol=2e-7)
    torch.testing.assert_close(g[:, vcol], want[:, vcol], rtol=2e-2, atol=2e-7)
    assert torch.all(g[:, S * A:vcol] == 0) and torch.all(g[:, vcol + 1:] == 0)
