// vy_ppo.cu — PPO rollout support kernels (config C3).
//
//   vy_gae: generalised advantage estimation as a reverse scan over the
//   rollout, one thread per env, [T][B] buffers (coalesced across envs at every
//   t).  delta_t = r_t + gamma * V_{t+1} * (1 - d_t) - V_t,
//   A_t = delta_t + gamma * lambda * (1 - d_t) * A_{t+1}, R_t = A_t + V_t
//   (PureJaxRL's formulation, which the paper's agent uses).
//
//   vy_ppo_sample: the multi-discrete policy head of the rollout in one pass —
//   Gumbel-max sampling of every slot's action from its logits and the
//   sample's log-probability (sum over slots of log softmax at the action).
//   vy_ppo_head_fwd / _bwd: the update's head — per-sample log-probability of
//   the stored actions and entropy (sum over slots), and the gradient of
//   g_lp * lp + g_ent * ent with respect to the logits, each one read of the
//   [N][S][A] logits (the unfused torch graph made ~10 passes over them).
//   One warp per sample, lanes over slots.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/voltyard_b200.h"

namespace {

__global__ void k_gae(const float* __restrict__ values, const float* __restrict__ rewards,
                      const uint8_t* __restrict__ dones, const float* __restrict__ last_value, int T, int64_t B,
                      float gamma, float lam, float* __restrict__ adv, float* __restrict__ ret) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float next_v = last_value[b];
  float gae = 0.f;
  for (int t = T - 1; t >= 0; --t) {
    const int64_t i = (int64_t)t * B + b;
    const float v = values[i];
    const float nonterm = dones[i] ? 0.f : 1.f;
    const float delta = rewards[i] + gamma * next_v * nonterm - v;
    gae = delta + gamma * lam * nonterm * gae;
    adv[i] = gae;
    ret[i] = gae + v;
    next_v = v;
  }
}

// per-slot softmax statistics of A logits: max, log-sum-exp
__device__ __forceinline__ void slot_lse(const float* __restrict__ z, int A, float& m, float& lse) {
  m = -INFINITY;
  for (int k = 0; k < A; ++k) m = fmaxf(m, z[k]);
  float sum = 0.f;
  for (int k = 0; k < A; ++k) sum += __expf(z[k] - m);
  lse = m + __logf(sum);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_ppo_sample(const float* __restrict__ logits, const float* __restrict__ noise, int64_t N, int S,
                             int A, uint8_t* __restrict__ actions, float* __restrict__ logp) {
  const int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float acc = 0.f;
  for (int s = lane; s < S; s += 32) {
    const float* z = logits + (n * S + s) * A;
    const float* u = noise + (n * S + s) * A;
    float m, lse;
    slot_lse(z, A, m, lse);
    int best = 0;
    float bv = -INFINITY;
    for (int k = 0; k < A; ++k) {
      const float g = -__logf(-__logf(fminf(fmaxf(u[k], 1e-20f), 1.f)));  // Gumbel(0, 1)
      const float v = z[k] + g;
      if (v > bv) {
        bv = v;
        best = k;
      }
    }
    actions[n * S + s] = (uint8_t)best;
    acc += z[best] - lse;
  }
  acc = warp_sum(acc);
  if (lane == 0) logp[n] = acc;
}

__global__ void k_ppo_head_fwd(const float* __restrict__ logits, const uint8_t* __restrict__ actions, int64_t N,
                               int S, int A, float* __restrict__ lp, float* __restrict__ ent) {
  const int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float alp = 0.f, aent = 0.f;
  for (int s = lane; s < S; s += 32) {
    const float* z = logits + (n * S + s) * A;
    float m, lse;
    slot_lse(z, A, m, lse);
    float h = 0.f;
    for (int k = 0; k < A; ++k) {
      const float l = z[k] - lse;
      h -= __expf(l) * l;
    }
    alp += z[actions[n * S + s]] - lse;
    aent += h;
  }
  alp = warp_sum(alp);
  aent = warp_sum(aent);
  if (lane == 0) {
    lp[n] = alp;
    ent[n] = aent;
  }
}

// d(g_lp * lp + g_ent * ent) / dz_k = g_lp (1[k = a] - p_k) - g_ent p_k (log p_k + H), H = slot entropy
__global__ void k_ppo_head_bwd(const float* __restrict__ logits, const uint8_t* __restrict__ actions, int64_t N,
                               int S, int A, const float* __restrict__ g_lp, const float* __restrict__ g_ent,
                               float* __restrict__ grad) {
  const int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  const float gl = g_lp ? g_lp[n] : 0.f, ge = g_ent ? g_ent[n] : 0.f;
  for (int s = lane; s < S; s += 32) {
    const float* z = logits + (n * S + s) * A;
    float* d = grad + (n * S + s) * A;
    float m, lse;
    slot_lse(z, A, m, lse);
    float h = 0.f;
    for (int k = 0; k < A; ++k) {
      const float l = z[k] - lse;
      h -= __expf(l) * l;
    }
    const int a = actions[n * S + s];
    for (int k = 0; k < A; ++k) {
      const float l = z[k] - lse, p = __expf(l);
      d[k] = gl * ((k == a ? 1.f : 0.f) - p) - ge * p * (l + h);
    }
  }
}

constexpr int kWarpsPerBlock = 8;
unsigned warp_grid(int64_t N) { return (unsigned)((N + kWarpsPerBlock - 1) / kWarpsPerBlock); }

}  // namespace

extern "C" int vy_ppo_sample(const float* logits, const float* noise, int64_t N, int32_t S, int32_t A,
                             uint8_t* actions, float* logp, void* stream) {
  if (!logits || !noise || !actions || !logp || N < 1 || S < 1 || A < 1 || A > 256) return VY_ERR_ARG;
  k_ppo_sample<<<warp_grid(N), kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(logits, noise, N, S, A, actions,
                                                                                logp);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_ppo_head_fwd(const float* logits, const uint8_t* actions, int64_t N, int32_t S, int32_t A,
                               float* lp, float* ent, void* stream) {
  if (!logits || !actions || !lp || !ent || N < 1 || S < 1 || A < 1) return VY_ERR_ARG;
  k_ppo_head_fwd<<<warp_grid(N), kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(logits, actions, N, S, A, lp, ent);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_ppo_head_bwd(const float* logits, const uint8_t* actions, int64_t N, int32_t S, int32_t A,
                               const float* g_lp, const float* g_ent, float* grad, void* stream) {
  if (!logits || !actions || !grad || N < 1 || S < 1 || A < 1) return VY_ERR_ARG;
  k_ppo_head_bwd<<<warp_grid(N), kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(logits, actions, N, S, A, g_lp,
                                                                                 g_ent, grad);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_gae(const float* values, const float* rewards, const uint8_t* dones, const float* last_value,
                      int32_t T, int64_t B, float gamma, float lam, float* adv, float* ret, void* stream) {
  if (!values || !rewards || !dones || !last_value || !adv || !ret || T < 1 || B < 1) return VY_ERR_ARG;
  const unsigned grid = (unsigned)((B + 255) / 256);
  k_gae<<<grid, 256, 0, (cudaStream_t)stream>>>(values, rewards, dones, last_value, T, B, gamma, lam, adv, ret);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}
