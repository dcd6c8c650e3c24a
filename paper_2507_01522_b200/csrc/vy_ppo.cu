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
//   Both: one thread per (sample, slot), whole rows staged per block.
//   vy_ppo_sample_rng draws the sampler's uniforms in the kernel (no noise
//   tensor), with a device call counter so graph replays need no host work.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
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
  // unrolled so each batch of steps' loads is in flight before the
  // recurrence reaches it (at 16 envs the scan is one dependent chain per env)
#pragma unroll 8
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

// GAE straight into the update's per-sample rows {old log-prob, value,
// advantage, return} (float4), the same recurrence and roundings as k_gae.
// Small rollouts (the paper's 1-16 envs): one block stages values, rewards
// and dones in shared memory with coalesced loads, threads b < B scan their
// env from shared memory, then the block writes the rows coalesced.
__global__ void __launch_bounds__(1024) k_gae_scal_small(const float* __restrict__ values,
                                                          const float* __restrict__ rewards,
                                                          const uint8_t* __restrict__ dones,
                                                          const float* __restrict__ last_value,
                                                          const float* __restrict__ logp, int T, int B, float gamma,
                                                          float lam, float4* __restrict__ scal) {
  extern __shared__ float gs[];
  const int n = T * B;
  float* sv = gs;
  float* sr = gs + n;  // rewards, then advantages in place
  uint8_t* sd = reinterpret_cast<uint8_t*>(gs + 2 * n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sv[i] = values[i];
    sr[i] = rewards[i];
    sd[i] = dones[i];
  }
  __syncthreads();
  if ((int)threadIdx.x < B) {
    const int b = threadIdx.x;
    float next_v = last_value[b];
    float gae = 0.f;
    for (int t = T - 1; t >= 0; --t) {
      const int i = t * B + b;
      const float v = sv[i];
      const float nonterm = sd[i] ? 0.f : 1.f;
      const float delta = sr[i] + gamma * next_v * nonterm - v;
      gae = delta + gamma * lam * nonterm * gae;
      sr[i] = gae;
      next_v = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = sv[i], a = sr[i];
    scal[i] = make_float4(logp[i], v, a, a + v);
  }
}

__global__ void k_gae_scal(const float* __restrict__ values, const float* __restrict__ rewards,
                           const uint8_t* __restrict__ dones, const float* __restrict__ last_value,
                           const float* __restrict__ logp, int T, int64_t B, float gamma, float lam,
                           float4* __restrict__ scal) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float next_v = last_value[b];
  float gae = 0.f;
#pragma unroll 8
  for (int t = T - 1; t >= 0; --t) {
    const int64_t i = (int64_t)t * B + b;
    const float v = values[i];
    const float nonterm = dones[i] ? 0.f : 1.f;
    const float delta = rewards[i] + gamma * next_v * nonterm - v;
    gae = delta + gamma * lam * nonterm * gae;
    scal[i] = make_float4(logp[i], v, gae, gae + v);
    next_v = v;
  }
}

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <class T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// The update's head runs on minibatches of ~300k samples, so it is laid out
// for bandwidth: a block stages G whole rows (G*ld values, contiguous in
// memory) with 16-byte loads, then one thread per (sample, slot) — G*S of
// the 256 threads, 255 for the 17-slot head — works on its slot's A values
// (slots A words apart: conflict-free for odd A), and per-sample sums go
// through shared memory.  The backward writes the gradient rows back the
// same way (padding columns zero).
constexpr int kHeadThreads = 256;

template <class T>
__device__ __forceinline__ void stage_rows(const T* __restrict__ src, int64_t n, float* __restrict__ dst) {
  constexpr int V = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && n % V == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll 4  // several vectors' loads in flight before the first conversion
    for (int64_t i = threadIdx.x; i < n / V; i += blockDim.x) {
      const uint4 u = __ldg(s4 + i);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int j = 0; j < V; ++j) dst[i * V + j] = to_f(e[j]);
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = to_f(src[i]);
  }
}

template <class T>
__device__ __forceinline__ void store_rows(const float* __restrict__ src, int64_t n, T* __restrict__ dst) {
  constexpr int V = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && n % V == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = threadIdx.x; i < n / V; i += blockDim.x) {
      uint4 u;
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int j = 0; j < V; ++j) e[j] = from_f<T>(src[i * V + j]);
      d4[i] = u;
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = from_f<T>(src[i]);
  }
}

// One slot's A logits: in registers when A is a compile-time constant AC
// (the 21-action head: one shared-memory read per logit instead of one per
// pass — the kernels were bound by shared-memory instructions), else read
// from the staged row.
template <int AC, class E = float>
struct Slot {
  float r[AC > 0 ? AC : 1];
  const E* p;
  int a;
  __device__ __forceinline__ Slot(const E* src, int A) : p(src), a(A) {
    if constexpr (AC > 0) {
#pragma unroll
      for (int k = 0; k < AC; ++k) r[k] = to_f(src[k]);
    }
  }
  __device__ __forceinline__ int size() const { return AC > 0 ? AC : a; }
  __device__ __forceinline__ float operator[](int k) const {
    if constexpr (AC > 0) return r[k];
    else return to_f(p[k]);
  }
};

// One slot's softmax statistics with a single exp per value: m = max z,
// e_k = exp(z_k - m), sum = sum e_k, logsum = log(sum), lse = m + logsum, and
// the entropy H = -sum p_k (z_k - lse) = logsum - sum(e_k (z_k - m)) / sum.
template <int AC, class E>
__device__ __forceinline__ void slot_stats(const Slot<AC, E>& z, float& m, float& logsum, float& inv, float& h) {
  m = -INFINITY;
#pragma unroll
  for (int k = 0; k < z.size(); ++k) m = fmaxf(m, z[k]);
  float sum = 0.f, ed = 0.f;
#pragma unroll
  for (int k = 0; k < z.size(); ++k) {
    const float d = z[k] - m, e = __expf(d);
    sum += e;
    ed += e * d;
  }
  inv = 1.f / sum;
  logsum = __logf(sum);
  h = logsum - ed * inv;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// n raw elements src -> dst (shared): 16-byte cp.async when both are aligned,
// else plain copies (complete on return)
template <class T>
__device__ __forceinline__ void issue_rows(const T* __restrict__ src, int64_t n, T* dst) {
  constexpr int V = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && n % V == 0) {
    for (int64_t i = threadIdx.x; i < n / V; i += blockDim.x) cp_async16(dst + i * V, src + i * V);
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

template <class T>
__host__ __device__ constexpr size_t raw_rows_bytes(int G, int64_t ld) {
  return ((size_t)G * ld * sizeof(T) + 15) & ~(size_t)15;
}

// Persistent and double-buffered: each block walks chunks of G rows
// (blockIdx.x, += gridDim.x) and copies the next chunk's raw rows into the
// other buffer with cp.async while it works on the current one, so the row
// loads overlap the softmax work (the one-chunk-per-block version stalled on
// them: long-scoreboard was its top stall).
template <class T, int AC>
__global__ void __launch_bounds__(kHeadThreads) k_ppo_head_fwd(const T* __restrict__ logits,
                                                               const uint8_t* __restrict__ actions, int64_t N, int S,
                                                               int A, int64_t ld, int G, float* __restrict__ lp,
                                                               float* __restrict__ ent) {
  extern __shared__ __align__(16) unsigned char ppo_raw[];
  const size_t rb = raw_rows_bytes<T>(G, ld);
  T* buf0 = reinterpret_cast<T*>(ppo_raw);
  T* buf1 = reinterpret_cast<T*>(ppo_raw + rb);
  float* part = reinterpret_cast<float*>(ppo_raw + 2 * rb);  // [2][G*S]
  const int64_t nch = (N + G - 1) / G;
  const int t = threadIdx.x;
  int64_t c = blockIdx.x;
  if (c < nch) issue_rows(logits + c * G * ld, (int64_t)min((int64_t)G, N - c * G) * ld, buf0);
  cp_async_commit();
  for (int i = 0; c < nch; c += gridDim.x, ++i) {
    const int64_t cn = c + gridDim.x;
    T* cur = (i & 1) ? buf1 : buf0;
    if (cn < nch) issue_rows(logits + cn * G * ld, (int64_t)min((int64_t)G, N - cn * G) * ld, (i & 1) ? buf0 : buf1);
    cp_async_commit();
    const int64_t n0 = c * G;
    const int gh = (int)min((int64_t)G, N - n0);
    const int act = t < gh * S ? actions[n0 * S + t] : 0;
    cp_async_wait<1>();  // every group but the one just issued: chunk c has landed
    __syncthreads();
    if (t < gh * S) {
      const int r = t / S, s = t - r * S;
      const T* zs = cur + (size_t)r * ld + s * A;
      const Slot<AC, T> z(zs, A);
      float m, logsum, inv, h;
      slot_stats(z, m, logsum, inv, h);
      part[t] = (to_f(zs[act]) - m) - logsum;
      part[G * S + t] = h;
    }
    __syncthreads();  // also frees `cur` for the copy issued next iteration
    if (t < gh) {
      float alp = 0.f, aent = 0.f;
      for (int s = 0; s < S; ++s) {
        alp += part[t * S + s];
        aent += part[G * S + t * S + s];
      }
      lp[n0 + t] = alp;
      ent[n0 + t] = aent;
    }
  }
  cp_async_wait<0>();
}

// d(g_lp * lp + g_ent * ent) / dz_k = g_lp (1[k = a] - p_k) - g_ent p_k (log p_k + H), H = slot entropy
template <class T, int AC>
__global__ void __launch_bounds__(kHeadThreads) k_ppo_head_bwd(const T* __restrict__ logits,
                                                               const uint8_t* __restrict__ actions, int64_t N, int S,
                                                               int A, int64_t ld, int G,
                                                               const float* __restrict__ g_lp,
                                                               const float* __restrict__ g_ent,
                                                               const float* __restrict__ g_value, int value_col,
                                                               T* __restrict__ grad) {
  // persistent and double-buffered like the forward; the gradient rows go
  // through a float32 staging area and leave with 16-byte stores
  extern __shared__ __align__(16) unsigned char ppo_raw[];
  const size_t rb = raw_rows_bytes<T>(G, ld);
  T* buf0 = reinterpret_cast<T*>(ppo_raw);
  T* buf1 = reinterpret_cast<T*>(ppo_raw + rb);
  float* out = reinterpret_cast<float*>(ppo_raw + 2 * rb);  // [G][ld]
  const int SA = S * A, pad = (int)(ld - SA);
  const int64_t nch = (N + G - 1) / G;
  const int t = threadIdx.x;
  int64_t c = blockIdx.x;
  if (c < nch) issue_rows(logits + c * G * ld, (int64_t)min((int64_t)G, N - c * G) * ld, buf0);
  cp_async_commit();
  for (int i = 0; c < nch; c += gridDim.x, ++i) {
    const int64_t cn = c + gridDim.x;
    T* cur = (i & 1) ? buf1 : buf0;
    if (cn < nch) issue_rows(logits + cn * G * ld, (int64_t)min((int64_t)G, N - cn * G) * ld, (i & 1) ? buf0 : buf1);
    cp_async_commit();
    const int64_t n0 = c * G;
    const int gh = (int)min((int64_t)G, N - n0);
    const bool live = t < gh * S;
    const int r = live ? t / S : 0, s = t - r * S;
    const int a = live ? actions[n0 * S + t] : 0;
    const float gl = live && g_lp ? g_lp[n0 + r] : 0.f, ge = live && g_ent ? g_ent[n0 + r] : 0.f;
    cp_async_wait<1>();
    __syncthreads();  // chunk c landed; the previous chunk's gradient rows have left `out`
    if (live) {
      const T* zs = cur + (size_t)r * ld + s * A;
      float* os = out + (size_t)r * ld + s * A;
      const Slot<AC, T> z(zs, A);
      float m, logsum, inv, h;
      slot_stats(z, m, logsum, inv, h);
#pragma unroll
      for (int k = 0; k < z.size(); ++k) {
        const float d = z[k] - m, p = __expf(d) * inv, l = d - logsum;
        os[k] = gl * ((k == a ? 1.f : 0.f) - p) - ge * p * (l + h);
      }
    }
    for (int j = t; j < gh * pad; j += blockDim.x) {  // padding columns: 0, or the value head's gradient
      const int rr = j / pad, col = SA + (j - rr * pad);
      out[(size_t)rr * ld + col] = (g_value && col == value_col) ? g_value[n0 + rr] : 0.f;
    }
    __syncthreads();
    store_rows(out, (int64_t)gh * ld, grad + n0 * ld);
  }
  cp_async_wait<0>();
}

// The whole PPO minibatch loss head in one pass over the logits: per
// sample the log-probability of the stored actions and the entropy (as
// k_ppo_head_fwd), the value from its padding column, the clipped surrogate,
// clipped value loss and entropy bonus (PPO; torch's
// min / max / clamp subgradients: ties split evenly, clamp bounds inclusive),
// and the gradient of
//   loss = mean(-min(r a, clip(r) a)) + vf_coef * mean(0.5 max((v-R)^2, (v_c-R)^2)) - ent_coef * mean(H)
// with respect to the logits rows (as k_ppo_head_bwd with the per-sample
// upstream gradients computed in place).  a = normalised advantage, from the
// minibatch mean / std in `adv_stats` (device).  Per-block partial sums of
// {loss, pg, vf, ent} (x N) go to `stats` with one atomic each per block.
struct LossCfg {
  float clip_eps, vf_clip, vf_coef, ent_coef;
};

template <class T, int AC>
__global__ void __launch_bounds__(kHeadThreads) k_ppo_loss(const T* __restrict__ logits,
                                                           const uint8_t* __restrict__ actions, int64_t N, int S,
                                                           int A, int64_t ld, int G, const float4* __restrict__ scal,
                                                           const float* __restrict__ adv_stats, LossCfg cfg,
                                                           int value_col, T* __restrict__ grad,
                                                           float* __restrict__ stats) {
  extern __shared__ __align__(16) unsigned char ppo_raw[];
  const size_t rb = raw_rows_bytes<T>(G, ld);
  T* buf0 = reinterpret_cast<T*>(ppo_raw);
  T* buf1 = reinterpret_cast<T*>(ppo_raw + rb);
  float* out = reinterpret_cast<float*>(ppo_raw + 2 * rb);  // [G][ld]
  float* part = out + (size_t)G * ld;                       // [2][G*S] slot partials
  float* gs = part + 2 * (size_t)G * S;                     // [3][G] per-sample g_lp, g_ent, g_v
  const int SA = S * A, pad = (int)(ld - SA);
  const int64_t nch = (N + G - 1) / G;
  const int t = threadIdx.x;
  const float inv_n = 1.f / (float)N;
  const float amean = adv_stats[0], astd = adv_stats[1];
  float acc_loss = 0.f, acc_pg = 0.f, acc_vf = 0.f, acc_ent = 0.f;  // samples of thread t (t < G)
  int64_t c = blockIdx.x;
  if (c < nch) issue_rows(logits + c * G * ld, (int64_t)min((int64_t)G, N - c * G) * ld, buf0);
  cp_async_commit();
  for (int i = 0; c < nch; c += gridDim.x, ++i) {
    const int64_t cn = c + gridDim.x;
    T* cur = (i & 1) ? buf1 : buf0;
    if (cn < nch) issue_rows(logits + cn * G * ld, (int64_t)min((int64_t)G, N - cn * G) * ld, (i & 1) ? buf0 : buf1);
    cp_async_commit();
    const int64_t n0 = c * G;
    const int gh = (int)min((int64_t)G, N - n0);
    const bool live = t < gh * S;
    const int r = live ? t / S : 0, s = t - r * S;
    const int a = live ? actions[n0 * S + t] : 0;
    float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < gh) sc = scal[n0 + t];
    cp_async_wait<1>();
    __syncthreads();  // chunk c landed; the previous chunk's gradient rows have left `out`
    // per (sample, slot): softmax statistics, log-probability of the action, entropy
    float m = 0.f, logsum = 0.f, inv = 0.f, h = 0.f;
    const T* zs = cur + (size_t)r * ld + s * A;
    if (live) {
      const Slot<AC, T> z(zs, A);
      slot_stats(z, m, logsum, inv, h);
      part[t] = (to_f(zs[a]) - m) - logsum;
      part[G * S + t] = h;
    }
    __syncthreads();
    // per sample: the loss terms and their gradients with respect to lp, H, v
    if (t < gh) {
      float lp = 0.f, ent = 0.f;
      for (int q = 0; q < S; ++q) {
        lp += part[t * S + q];
        ent += part[G * S + t * S + q];
      }
      const float v = to_f(cur[(size_t)t * ld + value_col]);
      const float old_lp = sc.x, old_v = sc.y, an = (sc.z - amean) / (astd + 1e-8f), ret = sc.w;
      const float ratio = expf(lp - old_lp);
      const float u = ratio * an;
      const float rc = fminf(fmaxf(ratio, 1.f - cfg.clip_eps), 1.f + cfg.clip_eps);
      const float cc = rc * an;
      const float pg = -fminf(u, cc);
      const bool inside = ratio >= 1.f - cfg.clip_eps && ratio <= 1.f + cfg.clip_eps;
      const float du = u < cc ? 1.f : (u > cc ? 0.f : 0.5f), dc = 1.f - du;
      const float g_lp = -(du + dc * (inside ? 1.f : 0.f)) * an * ratio * inv_n;
      const float dv = v - old_v;
      const float dvc = fminf(fmaxf(dv, -cfg.vf_clip), cfg.vf_clip);
      const float vc = old_v + dvc;
      const float e1 = (v - ret) * (v - ret), e2 = (vc - ret) * (vc - ret);
      const float vl = 0.5f * fmaxf(e1, e2);
      const float d1 = e1 > e2 ? 1.f : (e1 < e2 ? 0.f : 0.5f), d2 = 1.f - d1;
      const bool vin = dv >= -cfg.vf_clip && dv <= cfg.vf_clip;
      const float g_v = cfg.vf_coef * inv_n * (d1 * (v - ret) + d2 * (vc - ret) * (vin ? 1.f : 0.f));
      gs[t] = g_lp;
      gs[G + t] = -cfg.ent_coef * inv_n;
      gs[2 * G + t] = g_v;
      acc_pg += pg;
      acc_vf += vl;
      acc_ent += ent;
      acc_loss += pg + cfg.vf_coef * vl - cfg.ent_coef * ent;
    }
    __syncthreads();
    // per (sample, slot): d loss / d logits (k_ppo_head_bwd's formula)
    if (live) {
      const float gl = gs[r], ge = gs[G + r];
      float* os = out + (size_t)r * ld + s * A;
      const Slot<AC, T> z(zs, A);
#pragma unroll
      for (int k = 0; k < z.size(); ++k) {
        const float d = z[k] - m, p = __expf(d) * inv, l = d - logsum;
        os[k] = gl * ((k == a ? 1.f : 0.f) - p) - ge * p * (l + h);
      }
    }
    for (int j = t; j < gh * pad; j += blockDim.x) {  // padding columns: 0, or the value head's gradient
      const int rr = j / pad, col = SA + (j - rr * pad);
      out[(size_t)rr * ld + col] = col == value_col ? gs[2 * G + rr] : 0.f;
    }
    __syncthreads();
    store_rows(out, (int64_t)gh * ld, grad + n0 * ld);
  }
  cp_async_wait<0>();
  // the block's partial sums: threads 0..G-1 hold them (warp 0 when G <= 32)
  if (t < 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc_loss += __shfl_down_sync(0xffffffffu, acc_loss, o);
      acc_pg += __shfl_down_sync(0xffffffffu, acc_pg, o);
      acc_vf += __shfl_down_sync(0xffffffffu, acc_vf, o);
      acc_ent += __shfl_down_sync(0xffffffffu, acc_ent, o);
    }
    if (t == 0) {
      atomicAdd(stats, acc_loss);
      atomicAdd(stats + 1, acc_pg);
      atomicAdd(stats + 2, acc_vf);
      atomicAdd(stats + 3, acc_ent);
    }
  }
}

// Row gather with 16-byte vectors: a row's vectors go to consecutive threads
// (coalesced reads of each random row, fully coalesced writes).
// I = 32-bit element indices when the gathered block fits (cheap division).
template <class I>
__global__ void k_gather_rows(const uint4* __restrict__ src, I vpr, const int64_t* __restrict__ idx, I total,
                              uint4* __restrict__ dst) {
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const I r = i / vpr, v = i - r * vpr;
    dst[i] = __ldg(src + idx[r] * (int64_t)vpr + v);
  }
}

// Rollout sampling, laid out like the head: G rows staged per block, one
// thread per (sample, slot) takes argmax_k z_k + Gumbel_k and adds the
// action's log-probability; per-sample sums through shared memory.  Uniforms
// come from `noise` [N][S][A] or, when it is NULL, from the splitmix64 stream
// of (seed, call, element): call = counter[0], bumped by the last block to
// finish (counter[1] counts finished blocks), so a CUDA-graph replay draws
// fresh noise with no host involvement.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <class T, int AC>
__global__ void __launch_bounds__(kHeadThreads) k_ppo_sample(const T* __restrict__ logits,
                                                             const float* __restrict__ noise, uint64_t seed,
                                                             unsigned long long* counter, int64_t N, int S, int A,
                                                             int64_t ld, int G, uint8_t* __restrict__ actions,
                                                             float* __restrict__ logp, float* __restrict__ value,
                                                             int value_col) {
  extern __shared__ float ppo_smem[];
  const int64_t n0 = (int64_t)blockIdx.x * G;
  const int gh = (int)min((int64_t)G, N - n0);
  float* rows = ppo_smem;
  float* part = ppo_smem + (size_t)G * ld;
  stage_rows(logits + n0 * ld, (int64_t)gh * ld, rows);
  const uint64_t key = noise ? 0 : mix64(seed ^ mix64(counter[0] + 0x9E3779B97F4A7C15ULL));
  __syncthreads();
  const int t = threadIdx.x;
  if (t < gh * S) {
    const int r = t / S, s = t - r * S;
    const float* zs = rows + (size_t)r * ld + s * A;
    const Slot<AC> z(zs, A);
    float m, logsum, inv, h;
    slot_stats(z, m, logsum, inv, h);
    const int64_t e0 = ((n0 + r) * S + s) * A;
    int best = 0;
    float bv = -INFINITY;
#pragma unroll
    for (int k = 0; k < z.size(); ++k) {
      float u;
      if (noise) {
        u = fminf(fmaxf(noise[e0 + k], 1e-20f), 1.f);
      } else {
        // 23 bits: (x + 0.5) * 2^-23 is exact in float and lies in (0, 1), so
        // the double log stays finite (24 bits rounded the top draw to 1.0)
        u = ((float)(mix64(key + (uint64_t)(e0 + k) * 0x9E3779B97F4A7C15ULL) >> 41) + 0.5f) * (1.f / 8388608.f);
      }
      const float v = z[k] - __logf(-__logf(u));  // + Gumbel(0, 1)
      if (v > bv) {
        bv = v;
        best = k;
      }
    }
    actions[(n0 + r) * S + s] = (uint8_t)best;
    part[t] = (zs[best] - m) - logsum;
  }
  __syncthreads();
  if (t < gh) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += part[t * S + s];
    logp[n0 + t] = acc;
    if (value) value[n0 + t] = rows[(size_t)t * ld + value_col];  // a value head sharing the GEMM row
  }
  if (!noise && t == 0) {
    __threadfence();
    if (atomicAdd(counter + 1, 1ull) == gridDim.x - 1) {  // last block: every block has read counter[0]
      counter[1] = 0;
      counter[0] += 1;
      __threadfence();
    }
  }
}

// Column sums of a row-major [M][N] matrix (a linear layer's bias
// gradient) in two deterministic passes: each block of the first walks a
// band of rows with one thread per column (rows read whole and coalesced,
// eight loads in flight per thread) and writes its float32 partial sums to
// work[band][N]; the second adds the bands in order.  No atomics, so the
// result is the same on every run.
constexpr int kColsumBands = VY_COLSUM_BANDS;

template <class T>
__global__ void __launch_bounds__(512) k_colsum_bands(const T* __restrict__ g, int64_t M, int N, int64_t ld,
                                                      int64_t rows_per_band, float* __restrict__ work) {
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_band;
  const int64_t r1 = min(M, r0 + rows_per_band);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    float acc = 0.f;
    int64_t r = r0;
    for (; r + 8 <= r1; r += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = to_f(g[(r + j) * ld + c]);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
    for (; r < r1; ++r) acc += to_f(g[r * ld + c]);
    work[(int64_t)blockIdx.y * N + c] = acc;
  }
}

// bf16 rows with an even width: one thread per column pair (4-byte loads),
// half the load instructions of the per-column kernel
__global__ void __launch_bounds__(512) k_colsum_bands_bf2(const __nv_bfloat162* __restrict__ g, int64_t M, int N2,
                                                          int64_t ld2, int64_t rows_per_band, float* __restrict__ work) {
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_band;
  const int64_t r1 = min(M, r0 + rows_per_band);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N2; c += gridDim.x * blockDim.x) {
    float a0 = 0.f, a1 = 0.f;
    int64_t r = r0;
    for (; r + 8 <= r1; r += 8) {
      float2 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __bfloat1622float2(g[(r + j) * ld2 + c]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a0 += v[j].x;
        a1 += v[j].y;
      }
    }
    for (; r < r1; ++r) {
      const float2 v = __bfloat1622float2(g[r * ld2 + c]);
      a0 += v.x;
      a1 += v.y;
    }
    work[(int64_t)blockIdx.y * 2 * N2 + 2 * c] = a0;
    work[(int64_t)blockIdx.y * 2 * N2 + 2 * c + 1] = a1;
  }
}

// 32 columns per block, 32 band groups per column summed with eight loads
// in flight each, then the 32 group sums added in group order.
__global__ void __launch_bounds__(1024) k_colsum_reduce(const float* __restrict__ work, int bands, int N,
                                                        float* __restrict__ out) {
  __shared__ float grp[32][33];
  const int lane = threadIdx.x & 31, gi = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int per = (bands + 31) / 32, b0 = gi * per, b1 = min(bands, b0 + per);
  float acc = 0.f;
  if (c < N) {
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = work[(int64_t)(b + j) * N + c];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
    for (; b < b1; ++b) acc += work[(int64_t)b * N + c];
  }
  grp[gi][lane] = acc;
  __syncthreads();
  if (gi == 0 && c < N) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) t += grp[j][lane];
    out[c] = t;
  }
}

int head_rows(int S) { return S <= kHeadThreads ? kHeadThreads / S : 0; }
size_t head_smem(int S, int64_t ld) {
  const int G = head_rows(S);
  return (size_t)G * ld * sizeof(float) + 2 * (size_t)G * S * sizeof(float);
}
unsigned head_grid(int64_t N, int S) { return (unsigned)((N + head_rows(S) - 1) / head_rows(S)); }

}  // namespace

// dtype: 0 = float32 logits (and gradient), 1 = bfloat16
namespace {
int launch_sample(const void* logits, int32_t dtype, int64_t ld, const float* noise, uint64_t seed, int64_t* counter,
                  int64_t N, int32_t S, int32_t A, uint8_t* actions, float* logp, float* value, int32_t value_col,
                  void* stream) {
  if (!logits || !actions || !logp || N < 1 || S < 1 || A < 1 || A > 256 || (dtype != 0 && dtype != 1) ||
      head_rows(S) < 1 || ld < (int64_t)S * A || head_smem(S, ld) > 48 * 1024 ||
      (value && (value_col < S * A || value_col >= ld)))
    return VY_ERR_ARG;
  auto st = (cudaStream_t)stream;
  const int G = head_rows(S);
  auto ctr = reinterpret_cast<unsigned long long*>(counter);
  if (dtype == 0) {
    if (A == 21)
      k_ppo_sample<float, 21><<<head_grid(N, S), kHeadThreads, head_smem(S, ld), st>>>(
        static_cast<const float*>(logits), noise, seed, ctr, N, S, A, ld, G, actions, logp, value, value_col);
    else
      k_ppo_sample<float, 0><<<head_grid(N, S), kHeadThreads, head_smem(S, ld), st>>>(
        static_cast<const float*>(logits), noise, seed, ctr, N, S, A, ld, G, actions, logp, value, value_col);
  } else {
    if (A == 21)
      k_ppo_sample<__nv_bfloat16, 21><<<head_grid(N, S), kHeadThreads, head_smem(S, ld), st>>>(
        static_cast<const __nv_bfloat16*>(logits), noise, seed, ctr, N, S, A, ld, G, actions, logp, value, value_col);
    else
      k_ppo_sample<__nv_bfloat16, 0><<<head_grid(N, S), kHeadThreads, head_smem(S, ld), st>>>(
        static_cast<const __nv_bfloat16*>(logits), noise, seed, ctr, N, S, A, ld, G, actions, logp, value, value_col);
  }
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}
}  // namespace

extern "C" int vy_ppo_sample(const void* logits, int32_t dtype, int64_t ld, const float* noise, int64_t N, int32_t S,
                             int32_t A, uint8_t* actions, float* logp, void* stream) {
  if (!noise) return VY_ERR_ARG;
  return launch_sample(logits, dtype, ld, noise, 0, nullptr, N, S, A, actions, logp, nullptr, 0, stream);
}

extern "C" int vy_ppo_sample_rng(const void* logits, int32_t dtype, int64_t ld, uint64_t seed, int64_t* counter,
                                 int64_t N, int32_t S, int32_t A, uint8_t* actions, float* logp, float* value,
                                 int32_t value_col, void* stream) {
  if (!counter) return VY_ERR_ARG;
  return launch_sample(logits, dtype, ld, nullptr, seed, counter, N, S, A, actions, logp, value, value_col, stream);
}

extern "C" int vy_ppo_head_fwd(const void* logits, int32_t dtype, int64_t ld, const uint8_t* actions, int64_t N,
                               int32_t S, int32_t A, float* lp, float* ent, void* stream) {
  if (!logits || !actions || !lp || !ent || N < 1 || S < 1 || A < 1 || (dtype != 0 && dtype != 1) ||
      head_rows(S) < 1 || ld < (int64_t)S * A)
    return VY_ERR_ARG;
  auto st = (cudaStream_t)stream;
  const int G = head_rows(S);
  const size_t part = 2 * (size_t)G * S * sizeof(float);
  const size_t smem = (dtype == 0 ? 2 * raw_rows_bytes<float>(G, ld) : 2 * raw_rows_bytes<__nv_bfloat16>(G, ld)) + part;
  if (smem > 48 * 1024) return VY_ERR_ARG;
  const int64_t nch = (N + G - 1) / G;
  const unsigned grid = (unsigned)std::min<int64_t>(nch, 148 * 8);  // persistent: about one wave of resident blocks
  if (dtype == 0) {
    if (A == 21)
      k_ppo_head_fwd<float, 21><<<grid, kHeadThreads, smem, st>>>(static_cast<const float*>(logits), actions, N, S, A,
                                                                  ld, G, lp, ent);
    else
      k_ppo_head_fwd<float, 0><<<grid, kHeadThreads, smem, st>>>(static_cast<const float*>(logits), actions, N, S, A,
                                                                 ld, G, lp, ent);
  } else {
    if (A == 21)
      k_ppo_head_fwd<__nv_bfloat16, 21><<<grid, kHeadThreads, smem, st>>>(
          static_cast<const __nv_bfloat16*>(logits), actions, N, S, A, ld, G, lp, ent);
    else
      k_ppo_head_fwd<__nv_bfloat16, 0><<<grid, kHeadThreads, smem, st>>>(
          static_cast<const __nv_bfloat16*>(logits), actions, N, S, A, ld, G, lp, ent);
  }
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_ppo_head_bwd(const void* logits, int32_t dtype, int64_t ld, const uint8_t* actions, int64_t N,
                               int32_t S, int32_t A, const float* g_lp, const float* g_ent, const float* g_value,
                               int32_t value_col, void* grad, void* stream) {
  if (!logits || !actions || !grad || N < 1 || S < 1 || A < 1 || (dtype != 0 && dtype != 1) || head_rows(S) < 1 ||
      ld < (int64_t)S * A || (g_value && (value_col < S * A || value_col >= ld)))
    return VY_ERR_ARG;
  auto st = (cudaStream_t)stream;
  const int G = head_rows(S);
  const size_t smem = (dtype == 0 ? 2 * raw_rows_bytes<float>(G, ld) : 2 * raw_rows_bytes<__nv_bfloat16>(G, ld)) +
                      (size_t)G * ld * sizeof(float);
  if (smem > 200 * 1024) return VY_ERR_ARG;
  const int64_t nch = (N + G - 1) / G;
  const unsigned grid = (unsigned)std::min<int64_t>(nch, 148 * 8);
  if (smem > 48 * 1024) {  // float32 rows of the 17 x 21 head: 64 KB (opt-in above the 48 KB default)
    auto k = dtype == 0 ? (A == 21 ? (const void*)k_ppo_head_bwd<float, 21> : (const void*)k_ppo_head_bwd<float, 0>)
                        : (A == 21 ? (const void*)k_ppo_head_bwd<__nv_bfloat16, 21>
                                   : (const void*)k_ppo_head_bwd<__nv_bfloat16, 0>);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return VY_ERR_CUDA;
  }
  if (dtype == 0) {
    if (A == 21)
      k_ppo_head_bwd<float, 21><<<grid, kHeadThreads, smem, st>>>(static_cast<const float*>(logits), actions, N, S, A,
                                                                  ld, G, g_lp, g_ent, g_value, value_col, static_cast<float*>(grad));
    else
      k_ppo_head_bwd<float, 0><<<grid, kHeadThreads, smem, st>>>(static_cast<const float*>(logits), actions, N, S, A,
                                                                 ld, G, g_lp, g_ent, g_value, value_col, static_cast<float*>(grad));
  } else {
    if (A == 21)
      k_ppo_head_bwd<__nv_bfloat16, 21><<<grid, kHeadThreads, smem, st>>>(
          static_cast<const __nv_bfloat16*>(logits), actions, N, S, A, ld, G, g_lp, g_ent,
          g_value, value_col, static_cast<__nv_bfloat16*>(grad));
    else
      k_ppo_head_bwd<__nv_bfloat16, 0><<<grid, kHeadThreads, smem, st>>>(
          static_cast<const __nv_bfloat16*>(logits), actions, N, S, A, ld, G, g_lp, g_ent,
          g_value, value_col, static_cast<__nv_bfloat16*>(grad));
  }
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_gather_rows(const void* src, int64_t row_bytes, const int64_t* idx, int64_t n, void* dst,
                              void* stream) {
  if (n < 0 || row_bytes < 16 || row_bytes % 16) return VY_ERR_ARG;
  if (n == 0) return VY_OK;  // nothing to read or write (empty tensors may have null pointers)
  if (!src || !idx || !dst || (reinterpret_cast<uintptr_t>(src) & 15u) || (reinterpret_cast<uintptr_t>(dst) & 15u))
    return VY_ERR_ARG;
  const int64_t vpr = row_bytes / 16, total = n * vpr;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  auto st = (cudaStream_t)stream;
  // 32-bit indexing only when the grid-stride loop cannot wrap past 2^32
  // (idx values must lie in [0, rows of src); they are not bounds-checked)
  if (total + (int64_t)grid * 256 <= (int64_t)UINT32_MAX)
    k_gather_rows<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), (uint32_t)vpr, idx,
                                                  (uint32_t)total, static_cast<uint4*>(dst));
  else
    k_gather_rows<int64_t><<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), vpr, idx, total,
                                                 static_cast<uint4*>(dst));
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_colsum(const void* g, int32_t dtype, int64_t M, int64_t N, int64_t ld, float* work, float* out,
                         void* stream) {
  if (!out || !work || M < 0 || N < 1 || N > (1 << 20) || ld < N || (dtype != 0 && dtype != 1)) return VY_ERR_ARG;
  auto st = (cudaStream_t)stream;
  if (M == 0) {
    return cudaMemsetAsync(out, 0, (size_t)N * sizeof(float), st) == cudaSuccess ? VY_OK : VY_ERR_CUDA;
  }
  if (!g) return VY_ERR_ARG;
  const bool pairs = dtype == 1 && N % 2 == 0 && ld % 2 == 0 && (reinterpret_cast<uintptr_t>(g) & 3u) == 0;
  const int64_t cols = pairs ? N / 2 : N;  // threads' columns (pairs for even-width bf16)
  const int threads = cols >= 512 ? 512 : ((int)cols + 31) / 32 * 32;  // one x-block up to 512 columns
  const unsigned gx = (unsigned)((cols + threads - 1) / threads);
  // enough row bands to fill the GPU a few times over, at least 64 rows each
  int64_t bands = std::min<int64_t>(kColsumBands, std::max<int64_t>(1, 148 * 8 / (int64_t)gx));
  const int64_t rpb = std::max<int64_t>(64, (M + bands - 1) / bands);
  bands = (M + rpb - 1) / rpb;
  const dim3 grid(gx, (unsigned)bands);
  if (pairs)
    k_colsum_bands_bf2<<<grid, threads, 0, st>>>(static_cast<const __nv_bfloat162*>(g), M, (int)(N / 2), ld / 2, rpb,
                                                 work);
  else if (dtype == 0)
    k_colsum_bands<float><<<grid, threads, 0, st>>>(static_cast<const float*>(g), M, (int)N, ld, rpb, work);
  else
    k_colsum_bands<__nv_bfloat16><<<grid, threads, 0, st>>>(static_cast<const __nv_bfloat16*>(g), M, (int)N, ld, rpb,
                                                            work);
  k_colsum_reduce<<<(unsigned)((N + 31) / 32), 1024, 0, st>>>(work, (int)bands, (int)N, out);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_gae(const float* values, const float* rewards, const uint8_t* dones, const float* last_value,
                      int32_t T, int64_t B, float gamma, float lam, float* adv, float* ret, void* stream) {
  if (!values || !rewards || !dones || !last_value || !adv || !ret || T < 1 || B < 1) return VY_ERR_ARG;
  const unsigned grid = (unsigned)((B + 255) / 256);
  k_gae<<<grid, 256, 0, (cudaStream_t)stream>>>(values, rewards, dones, last_value, T, B, gamma, lam, adv, ret);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_gae_scal(const float* values, const float* rewards, const uint8_t* dones, const float* last_value,
                           const float* logp, int32_t T, int64_t B, float gamma, float lam, float* scal4,
                           void* stream) {
  if (!values || !rewards || !dones || !last_value || !logp || !scal4 || T < 1 || B < 1 ||
      (reinterpret_cast<uintptr_t>(scal4) & 15u))
    return VY_ERR_ARG;
  const int64_t n = (int64_t)T * B;
  const size_t smem = (size_t)n * 9 + 16;
  if (B <= 1024 && smem <= 160 * 1024) {
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_gae_scal_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024) != cudaSuccess)
      return VY_ERR_CUDA;
    k_gae_scal_small<<<1, 1024, smem, (cudaStream_t)stream>>>(values, rewards, dones, last_value, logp, T, (int)B,
                                                               gamma, lam, reinterpret_cast<float4*>(scal4));
  } else {
    k_gae_scal<<<(unsigned)((B + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        values, rewards, dones, last_value, logp, T, B, gamma, lam, reinterpret_cast<float4*>(scal4));
  }
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

extern "C" int vy_ppo_loss(const void* logits, int64_t ld, const uint8_t* actions, int64_t N, int32_t S, int32_t A,
                           const float* scal4, const float* adv_stats, float clip_eps, float vf_clip, float vf_coef,
                           float ent_coef, int32_t value_col, void* grad, float* stats, void* stream) {
  if (!logits || !actions || !scal4 || !adv_stats || !grad || !stats || N < 1 || S < 1 || A < 1 ||
      head_rows(S) < 1 || head_rows(S) > 32 || ld < (int64_t)S * A || value_col < S * A || value_col >= ld ||
      (reinterpret_cast<uintptr_t>(scal4) & 15u))
    return VY_ERR_ARG;
  auto st = (cudaStream_t)stream;
  const int G = head_rows(S);
  const size_t smem = 2 * raw_rows_bytes<__nv_bfloat16>(G, ld) + (size_t)G * ld * sizeof(float) +
                      (2 * (size_t)G * S + 3 * (size_t)G) * sizeof(float);
  if (smem > 200 * 1024) return VY_ERR_ARG;
  const int64_t nch = (N + G - 1) / G;
  const unsigned grid = (unsigned)std::min<int64_t>(nch, 148 * 8);
  auto k = A == 21 ? k_ppo_loss<__nv_bfloat16, 21> : k_ppo_loss<__nv_bfloat16, 0>;
  if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return VY_ERR_CUDA;
  const LossCfg cfg{clip_eps, vf_clip, vf_coef, ent_coef};
  k<<<grid, kHeadThreads, smem, st>>>(static_cast<const __nv_bfloat16*>(logits), actions, N, S, A, ld, G,
                                      reinterpret_cast<const float4*>(scal4), adv_stats, cfg, value_col,
                                      static_cast<__nv_bfloat16*>(grad), stats);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

namespace {
// x *= *g for bf16 x, unless *g == 1 (read on the device: no host sync; the
// unit upstream gradient of a loss that is the root of backward() costs one
// tiny launch)
__global__ void k_scale_bf16_unless_one(__nv_bfloat16* __restrict__ x, int64_t n, const float* __restrict__ g) {
  const float s = *g;
  if (s == 1.f) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __float2bfloat16_rn(__bfloat162float(x[i]) * s);
}
}  // namespace

extern "C" int vy_scale_bf16(void* x, int64_t n, const float* g, void* stream) {
  if (!x || !g || n < 0) return VY_ERR_ARG;
  if (n == 0) return VY_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_scale_bf16_unless_one<<<grid, 256, 0, (cudaStream_t)stream>>>(static_cast<__nv_bfloat16*>(x), n, g);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

namespace {
__device__ __forceinline__ uint64_t perm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// count pseudo-random permutations of 0..n-1 (the PPO update's minibatch
// shuffles): element i maps through a keyed 4-round Feistel bijection on
// [0, 4^h) (4^h >= n), cycle-walking until the image is < n — a bijection of
// [0, n) evaluated independently per element, no sort; each permutation has
// its own key from (seed, call, c).  The last CTA out advances the call counter.
__global__ void __launch_bounds__(256) k_random_perms(int64_t n, int h, uint64_t seed, unsigned long long* counter,
                                                       int64_t* __restrict__ out) {
  const int c = blockIdx.y;
  const uint64_t key = perm_mix(seed ^ perm_mix(counter[0] * 0x9E3779B97F4A7C15ULL + (uint64_t)c + 1));
  const uint32_t mask = (1u << h) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i;
    do {
      uint32_t L = x >> h, R = x & mask;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t f = (uint32_t)perm_mix(key + ((uint64_t)r << 40) + R) & mask;
        const uint32_t t = L ^ f;
        L = R;
        R = t;
      }
      x = (L << h) | R;
    } while ((int64_t)x >= n);
    out[(int64_t)c * n + i] = (int64_t)x;
  }
  __syncthreads();  // every thread of the CTA has read the call counter
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter + 1, 1ull) == gridDim.x * gridDim.y - 1) {
      counter[1] = 0;
      counter[0] += 1;
      __threadfence();
    }
  }
}
}  // namespace

extern "C" int vy_random_perms(int64_t n, int32_t count, uint64_t seed, int64_t* counter, int64_t* out,
                               void* stream) {
  if (!counter || !out || n < 1 || count < 1) return VY_ERR_ARG;
  if (n > (int64_t)1 << 30) return VY_ERR_UNSUPPORTED;
  int h = 1;
  while (((int64_t)1 << (2 * h)) < n) ++h;  // 4^h >= n: at most 4x the elements, ~2 walk steps on average
  const unsigned gx = (unsigned)std::min<int64_t>((n + 255) / 256, 1024);
  k_random_perms<<<dim3(gx, (unsigned)count), 256, 0, (cudaStream_t)stream>>>(
      n, h, seed, reinterpret_cast<unsigned long long*>(counter), out);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}
