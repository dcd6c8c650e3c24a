"""PPO on the device-resident env (BASELINE config C3).

The reference ships no trainer; the paper trains a PureJaxRL PPO
agent (hyperparameters PAPER.md:465-490).  This module is that
loop B200-first:

* rollout: per step ONE policy kernel (csrc/vy_policy.cu: the three MLP
  layers as tcgen05.mma on the 5th-generation tensor cores with TMEM
  accumulators, observation tiles bulk-copied by the TMA engine, tanh /
  bias epilogues and the categorical sampling of the 17 x 21 multi-discrete
  head fused) and the fused env step kernel, for T steps, captured once as a
  CUDA graph and replayed every iteration (fused_policy=False keeps the
  earlier cuBLAS + sampler-kernel path for comparison); at up to 4736 envs
  on lean stations the whole rollout is ONE kernel instead
  (csrc/vy_ppo_rollout.cuh: 16 envs per CTA, the same policy arithmetic and
  env step, weights and TMEM set up once for all T steps);
* advantages: the vy_gae reverse-scan kernel (csrc/vy_ppo.cu);
* update: clipped PPO objective with value clipping, entropy bonus, Adam,
  global-norm gradient clipping; under torch.distributed the flattened
  gradient is all-reduced (NCCL over NVLink) once per minibatch — the only
  data-path collective of the whole system.  Minibatches of <= 8192 samples
  (the paper's 1-16 env workloads) run as three kernels each
  (csrc/vy_ppo_update.cu: fp32 forward + loss + backward with per-CTA
  partial gradients, their ordered sum, clip + Adam in place) with the
  epochs' shuffles from one vy_random_perms launch; larger ones through
  autograd (bf16 GEMMs, the fused loss head, fused Adam).

Network: PureJaxRL's default actor-critic (two 64-unit tanh layers each for
actor and critic, orthogonal init); the paper does not pin the width, so it
is a constructor argument (recorded in the bench line).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist
import torch.nn as nn

from . import _native as nat
from .batch import BatchEnv


@dataclass
class PPOConfig:
    """PAPER.md:465-490 (Table 4)."""

    lr: float = 2.5e-4
    anneal_lr: bool = True
    gamma: float = 0.99
    gae_lambda: float = 0.95
    max_grad_norm: float = 100.0
    clip_eps: float = 0.2
    vf_clip: float = 10.0
    ent_coef: float = 0.01
    vf_coef: float = 0.25
    rollout_steps: int = 300
    n_minibatches: int = 4
    update_epochs: int = 4
    total_timesteps: int = 10_000_000
    hidden: int = 64
    seed: int = 0
    use_graph: bool = True
    fused_head: bool = True  # vy_ppo_sample / vy_ppo_head_* kernels instead of the torch op chain
    graph_update: bool = True  # the whole update (GAE + epochs x minibatches + Adam) as one CUDA graph (1 GPU)
    fused_policy: bool = True  # rollout forward + sampling in the tcgen05 kernel (vy_policy_step)
    # the whole rollout (policy passes + env steps) as one kernel at <= 4736 envs
    # (vy_ppo_rollout: up to 16 envs per CTA, at most two waves on 148 SMs:
    # 4096 envs 17.0 vs 25.0 us per step); lean stations without a battery,
    # else the per-step pair
    fused_rollout: bool = True
    # minibatches of <= 8192 samples: forward + loss + backward + clip + Adam as
    # three kernels per minibatch, fp32 (vy_ppo_update_*), instead of autograd
    fused_update: bool = True
    fused_loss: bool = True  # the update's loss head (log-prob, entropy, value, clipped losses, gradient) as one pass
    allreduce: str = "auto"  # gradient all-reduce: "auto" (world > 1), "always" (also at world 1: tests)
    wide_env: bool = True  # env step on the one-warp-per-env kernel at <= 2048 envs (vy_set_wide)


def _ortho(layer: nn.Linear, gain: float) -> nn.Linear:
    nn.init.orthogonal_(layer.weight, gain)
    nn.init.zeros_(layer.bias)
    return layer


def gather_rows(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """src[idx] for a row-major [n, w] tensor with 16-byte rows (vy_gather_rows;
    torch's indexing gathers these 224-byte rows at ~0.85 TB/s)."""
    row_bytes = src.shape[1] * src.element_size()
    if not (src.is_cuda and src.dim() == 2 and src.is_contiguous() and row_bytes % 16 == 0):
        raise ValueError("gather_rows needs a contiguous 2-D CUDA tensor with 16-byte-multiple rows")
    idx = idx.to(torch.int64).contiguous()
    out = torch.empty(idx.shape[0], src.shape[1], dtype=src.dtype, device=src.device)
    nat.check(nat.lib().vy_gather_rows(src.data_ptr(), row_bytes, idx.data_ptr(), idx.shape[0], out.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "vy_gather_rows")
    return out


def colsum(g: torch.Tensor) -> torch.Tensor:
    """Float32 column sums of a 2-D CUDA tensor (float32 / bf16, unit column
    stride) via vy_colsum: one pass at HBM rate, deterministic."""
    if g.dim() != 2 or g.stride(1) != 1:
        raise ValueError("colsum needs a 2-D tensor with unit column stride")
    out = torch.empty(g.shape[1], dtype=torch.float32, device=g.device)
    work = torch.empty(nat.COLSUM_BANDS, g.shape[1], dtype=torch.float32, device=g.device)
    nat.check(nat.lib().vy_colsum(g.data_ptr(), _dtype_code(g), g.shape[0], g.shape[1], g.stride(0),
                                  work.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream),
              "vy_colsum")
    return out


class _LinearFn(torch.autograd.Function):
    """y = x W^T + b whose backward forms the bias gradient with vy_colsum
    (one pass over the output gradient) instead of torch's sum(0), which ran
    2.5-4x slower on the update's ~300k-row minibatches
    (scripts/micro/bias_grad.py)."""

    @staticmethod
    @torch.amp.custom_fwd(device_type="cuda", cast_inputs=torch.bfloat16)
    def forward(ctx, x, w, b):
        ctx.save_for_backward(x, w)
        return nn.functional.linear(x, w, b)

    @staticmethod
    @torch.amp.custom_bwd(device_type="cuda")
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        g = g.contiguous()
        dx = g @ w if ctx.needs_input_grad[0] else None
        dw = g.t() @ x
        db = colsum(g).to(g.dtype)
        return dx, dw, db


class _Linear(nn.Linear):
    """nn.Linear with the GEMM bias gradient while training (2-D inputs); the
    plain layer otherwise, so inference keeps autocast's weight cache."""

    def forward(self, x):
        if torch.is_grad_enabled() and self.weight.requires_grad and x.dim() == 2 and x.is_cuda:
            return _LinearFn.apply(x, self.weight, self.bias)
        return super().forward(x)


def _ceil8(x: int) -> int:
    return (x + 7) // 8 * 8


class ActorCritic(nn.Module):
    """Actor-critic MLP.  The observation width (6n+9, odd) and the head width
    (S*A = 357) are padded to multiples of 8 — zero input columns, unused
    output columns — so the bf16 GEMMs have 16-byte aligned rows (cuBLAS
    otherwise falls back to sm75 kernels, 3-7x slower at these shapes,
    scripts/micro/gemm_align.py).  The actor's and the critic's first layers
    read the same observation, so they are one [2H x in] GEMM (rows 0..H-1
    actor, H..2H-1 critic; each half initialised as its own orthogonal layer):
    one pass over the observations and one launch instead of two."""

    def __init__(self, obs_dim: int, n_slots: int, n_actions: int, hidden: int = 64):
        super().__init__()
        self.n_slots, self.n_actions, self.hidden = n_slots, n_actions, hidden
        self.obs_dim, self.in_dim = obs_dim, _ceil8(obs_dim)
        self.n_out, self.out_dim = n_slots * n_actions, _ceil8(n_slots * n_actions)
        g = math.sqrt(2.0)
        self.inp = _Linear(self.in_dim, 2 * hidden)
        with torch.no_grad():
            for half in range(2):
                layer = _ortho(nn.Linear(self.in_dim, hidden), g)
                self.inp.weight[half * hidden:(half + 1) * hidden].copy_(layer.weight)
                self.inp.bias[half * hidden:(half + 1) * hidden].copy_(layer.bias)
        self.actor = nn.Sequential(_ortho(_Linear(hidden, hidden), g), nn.Tanh(),
                                   _ortho(_Linear(hidden, self.out_dim), 0.01))
        self.critic = nn.Sequential(_ortho(_Linear(hidden, hidden), g), nn.Tanh(),
                                    _ortho(_Linear(hidden, 1), 1.0))

    def pad_obs(self, obs: torch.Tensor) -> torch.Tensor:
        w = obs.shape[-1]
        return obs if w == self.in_dim else nn.functional.pad(obs, (0, self.in_dim - w))

    def forward(self, obs: torch.Tensor, logits_fp32: bool = True):
        """-> (logits, value).  logits_fp32: float32 [M, S, A] (torch head);
        else the raw padded head output [M, out_dim] (autocast dtype) that the
        fused head kernels read in place with row stride out_dim.  The value
        comes back in the compute dtype ([M]); callers widen it where they use it."""
        # split, not two slices: its backward is one concatenation of the two
        # halves' gradients (two slice backwards each write a zero-filled full width)
        ha, hc = torch.tanh(self.inp(self.pad_obs(obs))).split(self.hidden, dim=1)
        out = self.actor(ha)
        logits = out[:, : self.n_out].float().view(-1, self.n_slots, self.n_actions) if logits_fp32 else out
        return logits, self.critic(hc).squeeze(-1)

    def merged_weights(self) -> tuple:
        """Differentiable fp32 views of the second layers and heads as single
        matrices (see `inference_weights`): gradients flow back to the
        separate layers' parameters, the zero blocks get none."""
        H = self.hidden
        w2 = torch.block_diag(self.actor[0].weight, self.critic[0].weight)
        b2 = torch.cat([self.actor[0].bias, self.critic[0].bias])
        wh = torch.block_diag(self.actor[2].weight, self.critic[2].weight)  # [out_dim + 1, 2H]
        bh = torch.cat([self.actor[2].bias, self.critic[2].bias])
        pad = (-wh.shape[0]) % 8
        wh = nn.functional.pad(wh, (0, 0, 0, pad))
        bh = nn.functional.pad(bh, (0, pad))
        return w2, b2, wh, bh

    def forward_merged(self, x: torch.Tensor):
        """Training forward with three GEMMs (block-diagonal second layer,
        merged heads) on a padded input -> (head output [M, out_dim + 8]:
        logits in columns < out_dim, value in column out_dim; the value)."""
        w2, b2, wh, bh = self.merged_weights()
        lin = _LinearFn.apply if x.is_cuda else nn.functional.linear
        h = torch.tanh(self.inp(x))
        h = torch.tanh(lin(h, w2, b2))
        out = lin(h, wh, bh)
        return out, out[:, self.out_dim]

    @torch.no_grad()
    def inference_weights(self) -> tuple:
        """bf16 weights for `infer`, built once per rollout: the second layers
        as one block-diagonal [2H x 2H] matrix and the two heads as one
        [out_dim + 8 x 2H] matrix (actor rows, then the value row, zero-padded
        to a multiple of 8), so a policy step is three GEMMs instead of five."""
        H, bf = self.hidden, torch.bfloat16
        w2 = torch.block_diag(self.actor[0].weight, self.critic[0].weight)
        b2 = torch.cat([self.actor[0].bias, self.critic[0].bias])
        wh = torch.zeros(self.out_dim + 8, 2 * H, device=w2.device)
        wh[: self.out_dim, :H] = self.actor[2].weight
        wh[self.out_dim, H:] = self.critic[2].weight[0]
        bh = torch.zeros(self.out_dim + 8, device=w2.device)
        bh[: self.out_dim] = self.actor[2].bias
        bh[self.out_dim] = self.critic[2].bias[0]
        return (self.inp.weight.to(bf), self.inp.bias.to(bf), w2.to(bf), b2.to(bf), wh.to(bf), bh.to(bf))

    @torch.no_grad()
    def infer(self, x: torch.Tensor, w: tuple):
        """Rollout forward from `inference_weights` on a padded bf16 input ->
        (head output [M, out_dim + 8] bf16: logits in columns < out_dim, the
        value in column out_dim; the value column)."""
        f = nn.functional.linear
        h = torch.tanh(f(x, w[0], w[1]))
        h = torch.tanh(f(h, w[2], w[3]))
        out = f(h, w[4], w[5])
        return out, out[:, self.out_dim]


def policy_geometry(net: "ActorCritic", obs_ld: int | None = None) -> tuple[int, int, int, int]:
    """(weight blob bytes, float params, head rows, shared memory) of the
    tcgen05 policy kernel for this network (vy_policy_geometry)."""
    out = (C.c_int32 * 4)()
    rc = nat.lib().vy_policy_geometry(net.obs_dim, obs_ld or net.obs_dim, net.n_slots, net.n_actions, out)
    if rc != nat.VY_OK or net.hidden != 64:
        raise NotImplementedError("the tcgen05 policy kernel covers hidden=64, obs width <= 128, A <= 21")
    return tuple(out)


def _umma_k_major(w: torch.Tensor) -> torch.Tensor:
    """[N][K] -> the UMMA K-major no-swizzle layout [K/8][N][8] (bf16, flat)."""
    n, k = w.shape
    return w.to(torch.bfloat16).reshape(n, k // 8, 8).permute(1, 0, 2).reshape(-1)


def pack_policy(net: "ActorCritic", geo: tuple | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """The network's weights in the tcgen05 policy kernel's layout
    (csrc/vy_policy.cu): a bf16 blob [W1 | Wa2 | Wc2 | Wh] with every matrix
    in the UMMA K-major layout (W1 zero-padded to 16-column K steps; head row
    24s + k = logit k of slot s, the rest zero) and the float parameters
    b1, b2a, b2c, bh (same row map), wv, bv, each rounded through bf16 like
    the autocast forward's weights.  Differentiable ops on the live weights:
    call it inside a captured rollout so every replay uses the current ones."""
    geo = geo or policy_geometry(net)
    H, S, A = net.hidden, net.n_slots, net.n_actions
    dev = net.inp.weight.device
    k1 = (net.obs_dim + 15) // 16 * 16
    w1 = nn.functional.pad(net.inp.weight, (0, k1 - net.inp.weight.shape[1]))
    rows = (torch.arange(S, device=dev)[:, None] * 24 + torch.arange(A, device=dev)[None, :]).reshape(-1)
    wh = torch.zeros(geo[2], H, device=dev, dtype=net.inp.weight.dtype).index_copy(0, rows, net.actor[2].weight[: S * A])
    bh = torch.zeros(geo[2], device=dev, dtype=net.inp.weight.dtype).index_copy(0, rows, net.actor[2].bias[: S * A])
    blob = torch.cat([_umma_k_major(w1), _umma_k_major(net.actor[0].weight), _umma_k_major(net.critic[0].weight),
                      _umma_k_major(wh)])
    fp = torch.cat([net.inp.bias, net.actor[0].bias, net.critic[0].bias, bh, net.critic[2].weight[0],
                    net.critic[2].bias, torch.zeros(3, device=dev)])
    fp = fp.to(torch.bfloat16).float()
    assert blob.numel() * 2 == geo[0] and fp.numel() == geo[1]
    return blob, fp


def policy_step(obs: torch.Tensor, obs_dim: int, S: int, A: int, packed: tuple, seed: int, counter: torch.Tensor,
                actions: torch.Tensor, logp: torch.Tensor, value: torch.Tensor,
                logits_out: torch.Tensor | None = None) -> None:
    """One rollout step of the policy on the tensor cores (vy_policy_step):
    float32 obs rows [N, >= obs_dim] -> uint8 actions [N, S], log-probability
    and value [N] (float32), sampled with the device counter `counter`."""
    N = obs.shape[0]
    if obs.stride(1) != 1:
        raise ValueError("obs rows must be contiguous")
    blob, fp = packed
    rc = nat.lib().vy_policy_step(obs.data_ptr(), obs.stride(0), N, obs_dim, S, A, blob.data_ptr(), fp.data_ptr(),
                                  seed & ((1 << 64) - 1), counter.data_ptr(), actions.data_ptr(), logp.data_ptr(),
                                  value.data_ptr(), logits_out.data_ptr() if logits_out is not None else None,
                                  torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "vy_policy_step")


def ppo_rollout(env: BatchEnv, T: int, S: int, A: int, packed: tuple, seed: int, counter: torch.Tensor,
                obs: torch.Tensor, actions: torch.Tensor, logp: torch.Tensor, values: torch.Tensor,
                rewards: torch.Tensor, dones: torch.Tensor) -> None:
    """The whole rollout in one launch (vy_ppo_rollout): T x {tcgen05 policy
    pass + sampling, env step} and the bootstrap value, bit-identical to T + 1
    policy_step calls interleaved with T env.step calls.  obs [T+1, B, L]
    (row 0 read), actions [T, B, S], logp / rewards [T, B], values [T+1, B],
    dones [T, B]; all contiguous.  Raises NotImplementedError for stations the
    kernel does not cover (battery, > 32 ports)."""
    for t in (obs, actions, logp, values, rewards, dones):
        if not t.is_contiguous():
            raise ValueError("rollout buffers must be contiguous")
    blob, fp = packed
    rc = nat.lib().vy_ppo_rollout(env._h, int(T), blob.data_ptr(), fp.data_ptr(), S, A, seed & ((1 << 64) - 1),
                                  counter.data_ptr(), obs.data_ptr(), actions.data_ptr(), logp.data_ptr(),
                                  values.data_ptr(), rewards.data_ptr(), dones.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "vy_ppo_rollout")


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.bfloat16:
        return 1
    raise TypeError(f"logits must be float32 or bfloat16, got {t.dtype}")


class PolicyHead(torch.autograd.Function):
    """Per-sample log-probability of stored multi-discrete actions and entropy
    (both summed over slots) from logits rows of S x A values (float32 or
    bf16; row n starts at n * logits.stride(0), so the padded head output is
    read in place): vy_ppo_head_fwd / vy_ppo_head_bwd, one pass each way.
    With value_col >= 0 the rows also carry a value head in padding column
    value_col (the merged head GEMM): it is returned as a third output and its
    gradient is written by the same backward pass (a separate column select
    would add two full-width passes over the gradient)."""

    @staticmethod
    def forward(ctx, logits: torch.Tensor, actions: torch.Tensor, S: int, A: int, value_col: int = -1):
        N = logits.shape[0]
        ld = logits.stride(0)
        if logits.stride(-1) != 1 or logits[0].numel() < S * A or (logits.dim() > 2 and not logits[0].is_contiguous()):
            raise ValueError("logits rows must be contiguous with at least S*A values")
        if value_col >= 0 and not (S * A <= value_col < ld and logits.dim() == 2):
            raise ValueError("value_col must be a padding column of 2-D logits rows")
        lp = torch.empty(N, device=logits.device)
        ent = torch.empty(N, device=logits.device)
        nat.check(nat.lib().vy_ppo_head_fwd(logits.data_ptr(), _dtype_code(logits), ld, actions.data_ptr(), N, S, A,
                                            lp.data_ptr(), ent.data_ptr(), torch.cuda.current_stream().cuda_stream),
                  "vy_ppo_head_fwd")
        ctx.save_for_backward(logits, actions)
        ctx.S, ctx.A, ctx.value_col = S, A, value_col
        if value_col >= 0:
            return lp, ent, logits[:, value_col].float()
        return lp, ent

    @staticmethod
    def backward(ctx, g_lp, g_ent, g_v=None):
        logits, actions = ctx.saved_tensors
        N, S, A = logits.shape[0], ctx.S, ctx.A
        grad = torch.empty_like(logits)
        g_lp = g_lp.contiguous() if g_lp is not None else None
        g_ent = g_ent.contiguous() if g_ent is not None else None
        g_v = g_v.float().contiguous() if (g_v is not None and ctx.value_col >= 0) else None
        nat.check(nat.lib().vy_ppo_head_bwd(logits.data_ptr(), _dtype_code(logits), logits.stride(0),
                                            actions.data_ptr(), N, S, A,
                                            g_lp.data_ptr() if g_lp is not None else None,
                                            g_ent.data_ptr() if g_ent is not None else None,
                                            g_v.data_ptr() if g_v is not None else None, ctx.value_col,
                                            grad.data_ptr(), torch.cuda.current_stream().cuda_stream),
                  "vy_ppo_head_bwd")
        return grad, None, None, None, None


class PPOLoss(torch.autograd.Function):
    """The whole minibatch loss head as one pass (vy_ppo_loss): log-prob of
    the stored actions, entropy and value from the bf16 head rows, the
    clipped surrogate, clipped value loss and entropy bonus, and their
    gradient with respect to the head rows, all in the forward pass.  Returns
    the mean loss (differentiable) and the detached means (pg, vf, ent).  The
    backward scales the stored gradient by the upstream gradient on the
    device, in place (vy_scale_bf16: an early exit when it is 1, the loss
    being the root of ``backward()``, as in the trainer), so the graph is
    differentiated once (no ``retain_graph`` reuse)."""

    @staticmethod
    def forward(ctx, logits, actions, scal, adv_stats, S: int, A: int, value_col: int, clip_eps: float,
                vf_clip: float, vf_coef: float, ent_coef: float):
        if logits.dtype != torch.bfloat16 or logits.stride(-1) != 1 or logits.dim() != 2:
            raise ValueError("PPOLoss needs bf16 2-D head rows")
        N = logits.shape[0]
        grad = torch.empty_like(logits)
        stats = torch.zeros(4, device=logits.device)
        scal = scal.contiguous()
        nat.check(nat.lib().vy_ppo_loss(logits.data_ptr(), logits.stride(0), actions.data_ptr(), N, S, A,
                                        scal.data_ptr(), adv_stats.data_ptr(), clip_eps, vf_clip, vf_coef, ent_coef,
                                        value_col, grad.data_ptr(), stats.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream), "vy_ppo_loss")
        ctx.save_for_backward(grad)
        loss = stats[0] / N
        means = stats[1:] / N
        ctx.mark_non_differentiable(means)
        return loss, means

    @staticmethod
    def backward(ctx, g_loss, g_rest):
        (grad,) = ctx.saved_tensors
        g = g_loss.float().contiguous()
        nat.check(nat.lib().vy_scale_bf16(grad.data_ptr(), grad.numel(), g.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream), "vy_scale_bf16")
        return (grad,) + (None,) * 10


def head_reference(logits: torch.Tensor, actions: torch.Tensor):
    """Plain torch restatement of PolicyHead (tests only)."""
    lsm = torch.log_softmax(logits, dim=-1)
    lp = lsm.gather(-1, actions.long().unsqueeze(-1)).squeeze(-1).sum(-1)
    ent = -(lsm.exp() * lsm).sum(-1).sum(-1)
    return lp, ent


def allreduce_mean_(tensors: list, world: int, flat: torch.Tensor | None = None, group=None) -> None:
    """Average `tensors` over the ranks, in place: one flattened all-reduce
    (SUM, then / world — gloo has no AVG) instead of one per tensor.  `flat`
    (optional) is a preallocated buffer of the total size (graph capture:
    the same address every replay)."""
    n = sum(t.numel() for t in tensors)
    if flat is None:
        flat = torch.empty(n, dtype=tensors[0].dtype, device=tensors[0].device)
    off = 0
    for t in tensors:
        flat[off:off + t.numel()].copy_(t.reshape(-1))
        off += t.numel()
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    flat.div_(world)
    off = 0
    for t in tensors:
        t.copy_(flat[off:off + t.numel()].view_as(t))
        off += t.numel()


def gae(values, rewards, dones, last_value, gamma, lam):
    """Advantages and returns via the vy_gae kernel; [T, B] float32 / uint8 inputs."""
    T, B = values.shape
    adv = torch.empty_like(values)
    ret = torch.empty_like(values)
    rc = nat.lib().vy_gae(values.data_ptr(), rewards.data_ptr(), dones.data_ptr(), last_value.data_ptr(), T, B,
                          C.c_float(gamma), C.c_float(lam), adv.data_ptr(), ret.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "vy_gae")
    return adv, ret


def gae_reference(values, rewards, dones, last_value, gamma, lam):
    """Plain torch restatement (tests only)."""
    T = values.shape[0]
    adv = torch.zeros_like(values)
    last = torch.zeros_like(last_value)
    nxt = last_value
    for t in range(T - 1, -1, -1):
        nonterm = 1.0 - dones[t].float()
        delta = rewards[t] + gamma * nxt * nonterm - values[t]
        last = delta + gamma * lam * nonterm * last
        adv[t] = last
        nxt = values[t]
    return adv, adv + values


class PPOTrainer:
    """Single- or multi-GPU PPO over a BatchEnv (one process per GPU)."""

    def __init__(self, env: BatchEnv, cfg: PPOConfig):
        self.env, self.cfg = env, cfg
        dev = env.device
        if cfg.wide_env and env.batch_size <= 2048:
            # small batches: the tile step is latency-bound (a few warps on the
            # whole GPU); one warp per env, one lane per port steps in ~8 us
            # instead of ~14 (scripts/probe_step_small.py; at 4096 envs the
            # tile step is as fast and the wide one stops paying)
            env.set_wide(1)
        torch.manual_seed(cfg.seed + env.global_offset)
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.net = ActorCritic(env.obs_length, env.action_size, env.actions_per_slot, cfg.hidden).to(dev)
        if self.world > 1:  # identical initial weights on every rank
            for p in self.net.parameters():
                dist.broadcast(p.data, 0)
        # one graph replay per update (the update is launch-bound otherwise:
        # ~300 kernels per minibatch); under NCCL the per-minibatch gradient
        # all-reduce is captured in the same graph
        self._allreduce = self.world > 1 or cfg.allreduce == "always"
        nccl = dist.is_initialized() and dist.get_backend() == "nccl"
        self._graph_update = cfg.graph_update and cfg.use_graph and (not self._allreduce or nccl)
        if self._graph_update:
            self._lr = torch.tensor(cfg.lr, device=dev)
            self.opt = torch.optim.Adam(self.net.parameters(), lr=self._lr, eps=1e-5, fused=True, capturable=True)
        else:
            self.opt = torch.optim.Adam(self.net.parameters(), lr=cfg.lr, eps=1e-5, fused=True)
        self._ugraph = None
        self._ustats: dict = {}
        # rollout sampler stream: per-rank seed, {call, scratch} counter on the device
        self._sample_seed = (cfg.seed * 0x9E3779B1 + env.global_offset + 1) & ((1 << 64) - 1)
        self._sample_ctr = torch.zeros(2, dtype=torch.int64, device=dev)
        self._xin = torch.zeros(env.batch_size, self.net.in_dim, dtype=torch.bfloat16, device=dev)
        T, B, L, A = cfg.rollout_steps, env.batch_size, env.obs_length, env.action_size
        self.obs = torch.zeros(T + 1, B, L, device=dev)
        self.actions = torch.zeros(T, B, A, dtype=torch.uint8, device=dev)
        self.logp = torch.zeros(T, B, device=dev)
        self.values = torch.zeros(T + 1, B, device=dev)
        self.rewards = torch.zeros(T, B, device=dev)
        self.dones = torch.zeros(T, B, dtype=torch.uint8, device=dev)
        self.iterations = 0
        self.n_iters = max(1, cfg.total_timesteps // (T * B * self.world))
        self._graph = None
        self._fused_policy = cfg.fused_policy
        self._fused_rollout = cfg.fused_rollout and self._fused_policy and B <= 2 * 148 * 16
        if self._fused_policy:
            self._geo = policy_geometry(self.net)
            self._scratch_a = torch.zeros(B, A, dtype=torch.uint8, device=dev)
            self._scratch_lp = torch.zeros(B, device=dev)
        self._fused_update = False
        mb = T * B // cfg.n_minibatches
        if cfg.fused_update and cfg.hidden == 64 and 2 <= mb <= 8192:
            ws = (C.c_int64 * 4)()
            if nat.lib().vy_ppo_update_workspace(self.net.obs_dim, self.net.n_slots, self.net.n_actions, cfg.hidden,
                                                 mb, ws) == nat.VY_OK:
                self._fused_update = True
                P = ws[0]
                self._uwork = torch.zeros(ws[1], device=dev)
                self._ugrad = torch.zeros(P, device=dev)
                self._adam_m = torch.zeros(P, device=dev)
                self._adam_v = torch.zeros(P, device=dev)
                self._adam_step = torch.zeros(1, device=dev)
                self._ustats_buf = torch.zeros(4, device=dev)
                if not hasattr(self, "_lr"):
                    self._lr = torch.tensor(cfg.lr, device=dev)
                prm = list(self.net.parameters())
                assert sum(p.numel() for p in prm) == P
                self._uparams = (C.c_void_p * len(prm))(*[p.data_ptr() for p in prm])
                # W1 transposed for the first layer's coalesced reads (refreshed at
                # the start of every update, kept in step by the Adam kernel)
                self._uw1t = torch.empty(self.net.inp.weight.shape[1], self.net.inp.weight.shape[0], device=dev)
                # the epochs' minibatch shuffles in one launch (vy_random_perms, n <= 16384)
                self._perms = torch.empty(cfg.update_epochs, T * B, dtype=torch.int64, device=dev) \
                    if T * B <= 16384 else None
                self._perm_ctr = torch.zeros(2, dtype=torch.int64, device=dev)
                self._adv_stats = torch.zeros(cfg.update_epochs * cfg.n_minibatches, 2, device=dev)
                self._scal = torch.zeros(T * B, 4, device=dev)  # {old log-prob, value, advantage, return}
                self._perm_seed = (cfg.seed * 0x2545F4914F6CDD1D + env.global_offset + 7) & ((1 << 64) - 1)
        env.reset(as_numpy=False)
        self.obs[0].copy_(env.outs.obs)

    # -- rollout -----------------------------------------------------------------

    def _policy_step(self, t: int) -> None:
        if self._fused_policy:
            # obs -> 3 tcgen05 GEMM layers -> sampled actions / log-prob / value, one kernel
            policy_step(self.obs[t], self.env.obs_length, self.net.n_slots, self.net.n_actions, self._packed,
                        self._sample_seed, self._sample_ctr, self.actions[t], self.logp[t], self.values[t])
            self.env.set_outputs(obs=self.obs[t + 1], reward=self.rewards[t], done=self.dones[t])
            self.env.step(self.actions[t], collect_infos=False)
            return
        fused = self.cfg.fused_head
        # the padded bf16 network input in one copy (the zero padding columns of
        # the persistent buffer are never written): no pad + cast pair per step
        self._xin[:, : self.env.obs_length].copy_(self.obs[t])
        if fused:
            logits, v = self.net.infer(self._xin, self._iw)  # row stride out_dim + 8, read in place
        else:
            logits, v = self.net(self._xin, logits_fp32=True)
        if fused:
            # Gumbel-max sampling (uniforms drawn in the kernel, call counter on
            # the device) + log-probability in one kernel, into the rollout buffers
            B, S, A = logits.shape[0], self.net.n_slots, self.net.n_actions
            nat.check(nat.lib().vy_ppo_sample_rng(logits.data_ptr(), _dtype_code(logits), logits.stride(0),
                                                  self._sample_seed, self._sample_ctr.data_ptr(), B, S, A,
                                                  self.actions[t].data_ptr(), self.logp[t].data_ptr(),
                                                  self.values[t].data_ptr(), self.net.out_dim,  # value column too
                                                  torch.cuda.current_stream().cuda_stream), "vy_ppo_sample_rng")
        else:
            noise = torch.rand(logits.shape[0], self.net.n_slots, self.net.n_actions, device=logits.device)
            g = -torch.log(-torch.log(noise.clamp_(1e-20, 1.0)))  # Gumbel-max sampling
            a = torch.argmax(logits + g, dim=-1)
            lp = torch.log_softmax(logits, dim=-1).gather(-1, a.unsqueeze(-1)).squeeze(-1).sum(-1)
            self.actions[t].copy_(a)
            self.logp[t].copy_(lp)
            self.values[t].copy_(v)
        # the env writes the next obs / reward / done straight into the rollout buffers
        self.env.set_outputs(obs=self.obs[t + 1], reward=self.rewards[t], done=self.dones[t])
        self.env.step(self.actions[t], collect_infos=False)

    def _rollout_body(self) -> None:
        # one autocast region for the whole rollout: the bf16 copies of the
        # weights are made once per rollout (autocast's weight cache), not once
        # per policy step
        if self._fused_policy:
            self._packed = pack_policy(self.net, self._geo)  # inside the graph: from the live weights each replay
            if self._fused_rollout:
                try:
                    ppo_rollout(self.env, self.cfg.rollout_steps, self.net.n_slots, self.net.n_actions, self._packed,
                                self._sample_seed, self._sample_ctr, self.obs, self.actions, self.logp, self.values,
                                self.rewards, self.dones)
                    return
                except NotImplementedError:  # decided on the first (uncaptured) rollout
                    self._fused_rollout = False
            for t in range(self.cfg.rollout_steps):
                self._policy_step(t)
            # bootstrap value of the last obs (its actions / log-prob land in scratch rows)
            T = self.cfg.rollout_steps
            policy_step(self.obs[T], self.env.obs_length, self.net.n_slots, self.net.n_actions, self._packed,
                        self._sample_seed, self._sample_ctr, self._scratch_a, self._scratch_lp, self.values[T])
            return
        with torch.autocast("cuda", dtype=torch.bfloat16):
            if self.cfg.fused_head:
                self._iw = self.net.inference_weights()  # inside the graph: rebuilt from the live weights each replay
            for t in range(self.cfg.rollout_steps):
                self._policy_step(t)
            self._xin[:, : self.env.obs_length].copy_(self.obs[-1])
            _, v = self.net(self._xin)
            self.values[-1].copy_(v)

    @torch.no_grad()
    def rollout(self) -> None:
        T = self.cfg.rollout_steps
        t0 = self.env._t
        executed = 1  # rollouts the GPU runs in this call
        if not self.cfg.use_graph:
            self._rollout_body()
        else:
            if self._graph is None:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):  # warm-up outside capture (allocator, autocast caches)
                    self._rollout_body()
                torch.cuda.current_stream().wait_stream(s)
                self.obs[0].copy_(self.obs[-1])
                self._graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._graph):  # captured, not executed (env.step still ticks the host clock)
                    self._rollout_body()
                executed = 2  # the warm-up rollout, then the first replay below
            self._graph.replay()
        if t0 is not None:  # the host mirror of the lockstep clock: a graph replay runs no host code
            self.env._t = (t0 + executed * T) % self.env.tables.episode_steps
        self.env.restore_outputs()

    # -- update -------------------------------------------------------------------

    def _allreduce_grads(self) -> None:
        """Mean of the minibatch gradients over the ranks (NCCL over NVLink):
        the only data-path collective of the system, once per minibatch."""
        if not self._allreduce:
            return
        grads = [p.grad for p in self.net.parameters()]
        if getattr(self, "_flat_grad", None) is None:
            self._flat_grad = torch.empty(sum(g.numel() for g in grads), device=grads[0].device)
        allreduce_mean_(grads, self.world, self._flat_grad)

    def update(self) -> dict:
        cfg = self.cfg
        lr = cfg.lr * max(1.0 - self.iterations / self.n_iters, 0.0) if cfg.anneal_lr else cfg.lr
        if not self._graph_update:
            for g in self.opt.param_groups:
                g["lr"] = lr
            if self._fused_update:
                self._lr.fill_(lr)
            stats = self._update_body()
        else:
            self._lr.fill_(lr)
            if self._ugraph is None:
                cur = torch.cuda.current_stream()
                s = torch.cuda.Stream()
                s.wait_stream(cur)
                with torch.cuda.stream(s):  # this iteration's update, eager (warms up autograd / cuBLAS)
                    stats = self._update_body()
                cur.wait_stream(s)
                self._ugraph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._ugraph):  # captured, not executed
                    self._ustats = self._update_body()
            else:
                self._ugraph.replay()
                stats = {k: v.clone() for k, v in self._ustats.items()}
        self.iterations += 1
        return stats

    def _update_body(self) -> dict:
        cfg = self.cfg
        T, B = cfg.rollout_steps, self.env.batch_size
        if self._fused_update:
            return self._fused_update_body(T * B, T * B // cfg.n_minibatches)
        adv, ret = gae(self.values[:T], self.rewards, self.dones, self.values[T], cfg.gamma, cfg.gae_lambda)
        # aligned bf16 rows once per update (the value autocast would cast each
        # minibatch to anyway); minibatches gather half the bytes
        obs = self.net.pad_obs(self.obs[:T].reshape(T * B, -1)).to(torch.bfloat16)
        act = self.actions.reshape(T * B, -1)
        # the four per-sample scalars side by side: one 16-byte-row gather per minibatch
        scal = torch.stack([self.logp.reshape(-1), self.values[:T].reshape(-1), adv.reshape(-1), ret.reshape(-1)], 1)
        n = T * B
        mb = n // cfg.n_minibatches
        stats = {}
        for _ in range(cfg.update_epochs):
            perm = torch.argsort(torch.rand(n, device=obs.device))  # a uniform permutation, capture-safe
            for k in range(cfg.n_minibatches):
                idx = perm[k * mb:(k + 1) * mb]
                with torch.autocast("cuda", dtype=torch.bfloat16):
                    if cfg.fused_head:  # head output read in place by the fused head (row stride out_dim + 8)
                        logits, _ = self.net.forward_merged(gather_rows(obs, idx))
                    else:
                        logits, v = self.net(gather_rows(obs, idx), logits_fp32=True)
                        v = v.float()
                if cfg.fused_head and cfg.fused_loss and logits.dtype == torch.bfloat16:
                    # one pass: log-prob, entropy, value, clipped losses and d loss / d head rows
                    sc = gather_rows(scal, idx)
                    a = sc[:, 2]
                    adv_stats = torch.stack([a.mean(), a.std()])
                    loss, means = PPOLoss.apply(logits, act[idx], sc, adv_stats, self.net.n_slots, self.net.n_actions,
                                                self.net.out_dim, cfg.clip_eps, cfg.vf_clip, cfg.vf_coef,
                                                cfg.ent_coef)
                    self.opt.zero_grad(set_to_none=False)
                    loss.backward()
                    self._allreduce_grads()
                    nn.utils.clip_grad_norm_(self.net.parameters(), cfg.max_grad_norm)
                    self.opt.step()
                    stats = {"loss": loss.detach(), "pg": means[0], "vf": means[1], "ent": means[2]}
                    continue
                if cfg.fused_head:  # the value column rides through the head kernels too
                    lp, ent, v = PolicyHead.apply(logits, act[idx], self.net.n_slots, self.net.n_actions,
                                                  self.net.out_dim)
                else:
                    lp, ent = head_reference(logits, act[idx])
                ent = ent.mean()
                old_lp, old_v, a, r = gather_rows(scal, idx).unbind(1)
                a = (a - a.mean()) / (a.std() + 1e-8)
                ratio = torch.exp(lp - old_lp)
                pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip_eps, 1 + cfg.clip_eps) * a).mean()
                v_clip = old_v + (v - old_v).clamp(-cfg.vf_clip, cfg.vf_clip)
                vl = 0.5 * torch.max((v - r) ** 2, (v_clip - r) ** 2).mean()
                loss = pg + cfg.vf_coef * vl - cfg.ent_coef * ent
                self.opt.zero_grad(set_to_none=False)
                loss.backward()
                self._allreduce_grads()
                nn.utils.clip_grad_norm_(self.net.parameters(), cfg.max_grad_norm)
                self.opt.step()
                stats = {"loss": loss.detach(), "pg": pg.detach(), "vf": vl.detach(), "ent": ent.detach()}
        self.obs[0].copy_(self.obs[T])
        return stats

    def _fused_update_body(self, n: int, mb: int) -> dict:
        """GAE into the per-sample rows (vy_gae_scal), then epochs x
        minibatches of vy_ppo_update_grad (+ the gradient all-reduce across
        ranks) + vy_ppo_update_adam; the rollout rows are read in place through
        each minibatch's index slice."""
        cfg, T = self.cfg, self.cfg.rollout_steps
        lib, st = nat.lib(), torch.cuda.current_stream().cuda_stream
        obs = self.obs[:T].reshape(n, -1)
        act = self.actions.reshape(n, -1)
        scal = self._scal
        nat.check(lib.vy_gae_scal(self.values.data_ptr(), self.rewards.data_ptr(), self.dones.data_ptr(),
                                  self.values[T].data_ptr(), self.logp.data_ptr(), T, self.env.batch_size,
                                  C.c_float(cfg.gamma), C.c_float(cfg.gae_lambda), scal.data_ptr(), st),
                  "vy_gae_scal")
        S, A, H, od = self.net.n_slots, self.net.n_actions, cfg.hidden, self.net.obs_dim
        with torch.no_grad():
            self._uw1t.copy_(self.net.inp.weight.t())
        if self._perms is not None:  # the shuffles and every minibatch's advantage mean / std, two launches
            nat.check(lib.vy_random_perms(n, cfg.update_epochs, self._perm_seed, self._perm_ctr.data_ptr(),
                                          self._perms.data_ptr(), st), "vy_random_perms")
            nat.check(lib.vy_ppo_adv_stats(scal.data_ptr(), self._perms.data_ptr(), n, cfg.update_epochs,
                                           cfg.n_minibatches, mb, self._adv_stats.data_ptr(), st), "vy_ppo_adv_stats")
        for ep in range(cfg.update_epochs):
            if self._perms is not None:
                perm = self._perms[ep]
            else:
                perm = torch.argsort(torch.rand(n, device=obs.device))  # a uniform permutation, capture-safe
            for k in range(cfg.n_minibatches):
                idx = perm[k * mb:(k + 1) * mb]
                nat.check(lib.vy_ppo_update_grad(self._uparams, self._uw1t.data_ptr(), od, S, A, H, obs.data_ptr(), obs.stride(0),
                                                 act.data_ptr(), scal.data_ptr(), idx.data_ptr(),
                                                 self._adv_stats[ep * cfg.n_minibatches + k].data_ptr()
                                                 if self._perms is not None else None, mb, cfg.clip_eps,
                                                 cfg.vf_clip, cfg.vf_coef, cfg.ent_coef, self._uwork.data_ptr(),
                                                 self._ugrad.data_ptr(), self._ustats_buf.data_ptr(),
                                                 self._adam_step.data_ptr(), st), "vy_ppo_update_grad")
                if self._allreduce:  # the flat gradient, SUM then / world (gloo has no AVG)
                    dist.all_reduce(self._ugrad, op=dist.ReduceOp.SUM)
                    self._ugrad.div_(self.world)
                nat.check(lib.vy_ppo_update_adam(self._uparams, self._uw1t.data_ptr(), od, S, A, H, mb, self._uwork.data_ptr(),
                                                 self._ugrad.data_ptr(), self._adam_m.data_ptr(),
                                                 self._adam_v.data_ptr(), self._lr.data_ptr(),
                                                 self._adam_step.data_ptr(), 0.9, 0.999, 1e-5, cfg.max_grad_norm, st),
                          "vy_ppo_update_adam")
        self.obs[0].copy_(self.obs[T])
        s = self._ustats_buf
        return {"loss": s[0].clone(), "pg": s[1].clone(), "vf": s[2].clone(), "ent": s[3].clone()}

    def describe_update(self) -> str:
        if self._fused_update:
            return ("per minibatch: vy_ppo_update_grad (fp32 forward, clipped loss, backward, per-CTA partial "
                    "gradients; 8 or 16 samples per CTA, second layers and head staged in shared memory) + k_ppo_gsum (ordered sum, squares) + vy_ppo_update_adam "
                    "(clip_grad_norm_ + Adam in place); the epochs' shuffles in one vy_random_perms launch; epochs x "
                    "minibatches in one CUDA graph")
        return ("one CUDA graph per update: vy_gae, vy_gather_rows minibatch gather, bf16 GEMMs with column-sum "
                "bias gradients (vy_colsum), vy_ppo_loss, fused Adam")

    def describe_rollout(self) -> str:
        if self._fused_rollout:
            return ("one kernel per rollout: vy_ppo_rollout (per CTA 2-16 envs x T steps: tcgen05 3-layer MLP, TMEM "
                    "accumulators, fused epilogues + inverse-CDF sampling, then the one-warp-per-env step; weights, "
                    "TMEM and station tables set up once) + pack_policy")
        if self._fused_policy:
            return ("CUDA graph x T: vy_policy_step (tcgen05 3-layer MLP, TMEM accumulators, bulk-async obs tiles, "
                    "fused tanh/bias epilogues + inverse-CDF sampling, log-prob, value) + k_step")
        return ("CUDA graph x T: cuBLAS bf16 GEMMs (block-diagonal layer 2, merged heads) + vy_ppo_sample_rng "
                "Gumbel-max kernel + k_step")

    def iterate(self) -> dict:
        self.rollout()
        return self.update()


def seconds_per_100k(trainer: PPOTrainer, iters: int, warmup: int = 1) -> dict:
    """Wall-clock (device-synchronised) seconds per 100k env steps of rollout + update."""
    for _ in range(warmup):
        trainer.iterate()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    t0 = time.perf_counter()
    rewards = []
    for _ in range(iters):
        trainer.iterate()
        rewards.append(trainer.rewards.mean())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if dist.is_initialized():
        t = torch.tensor([dt], device=trainer.env.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    steps = iters * trainer.cfg.rollout_steps * trainer.env.batch_size * trainer.world
    return {"s_per_100k_steps": dt / steps * 1e5, "env_steps_per_s": steps / dt, "iters": iters,
            "mean_step_reward": float(torch.stack(rewards).mean()) if rewards else float("nan"),
            "seconds": dt, "steps": steps}


__all__ = ["PPOConfig", "ActorCritic", "PPOTrainer", "PolicyHead", "head_reference", "gae", "gae_reference",
           "seconds_per_100k", "np"]
