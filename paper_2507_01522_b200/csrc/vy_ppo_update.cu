// vy_ppo_update.cu — one PPO minibatch update (forward, clipped loss,
// backward, global-norm clipping, Adam) in three kernel launches, for the
// small batches the paper trains on (PPO(16): 1200-sample minibatches).
//
// The autograd path (ppo.py _update_body) is ~70 launches per minibatch —
// weight casts, three GEMM pairs, bias column sums, tanh forward/backward,
// the loss kernel, the norm, Adam — each a few microseconds of latency on an
// idle GPU at these sizes (~190 us per minibatch, CUDA graph replayed).  Here:
//   k_ppo_grad  (ceil(M/16) CTAs x 256 threads): every CTA normalises the
//     minibatch's advantages (mean / unbiased std over all M rows, the same
//     fixed-order reduction in every CTA), gathers its <= 16 rows, runs the
//     actor-critic forward in fp32 from the live fp32 weights (L2-resident),
//     the loss head of k_ppo_loss (same formulas: log-softmax per slot,
//     entropy, clipped surrogate, clipped value loss), the backward through
//     the three layers, and writes its partial weight gradient (sum over its
//     rows) and loss sums;
//   k_ppo_gsum  (one thread per parameter): the partials summed over the CTAs
//     in CTA order (deterministic) -> the flat gradient; per-block sums of
//     squares; block 0 also sums the loss statistics and advances the Adam
//     step counter;
//   (the caller may all-reduce the flat gradient here: NCCL, multi-GPU)
//   k_ppo_adam  (one thread per parameter): the global norm from the block
//     sums (fixed order), torch's clip_grad_norm_ coefficient
//     min(1, max_norm / (norm + 1e-6)), then torch's Adam (bias-corrected
//     moments, eps outside the square root) on the parameters in place.
// fp32 throughout (the autograd path runs bf16 autocast GEMMs): tests compare
// the gradient with torch fp32 autograd and the Adam step with torch's.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/voltyard_b200.h"

namespace vyu {

constexpr int kRows = 16;      // rows per CTA
constexpr int kThreads = 256;
constexpr int kH = 64;         // hidden width per branch
constexpr int kNP = 10;        // parameter tensors (ActorCritic order)

struct Net {
  const float* w[kNP];  // w1, b1, wa2, ba2, wh, bh, wc2, bc2, wv, bv
  int64_t off[kNP + 1];  // flat offsets (the module's parameter order)
  int K1, NO;            // padded input width (W1 columns), head rows (out_dim)
};

struct Batch {
  const float* obs;  // [*][obs_ld] float32 rollout rows
  int64_t obs_ld;
  int obs_dim;
  const uint8_t* actions;  // [*][S]
  const float4* scal;      // [*] {old_lp, old_v, adv, ret}
  const int64_t* idx;      // [M] rows of this minibatch
  int64_t M;
  int S, A;
  float clip_eps, vf_clip, vf_coef, ent_coef;
};

struct Work {
  float* part;   // [grid][P] per-CTA gradient partials
  float* lstat;  // [grid][4] per-CTA loss sums {loss, pg, vf, ent}
  float* grad;   // [P] flat gradient
  float* sq;     // [gsum blocks] sums of squares
  float* stats;  // [4] minibatch means {loss, pg, vf, ent}
  float* step;   // Adam step counter (float, on the device)
};

__device__ __forceinline__ float block_sum(float v, float* red) {
  // fixed-order block reduction (warp shuffles, then warp 0 over the warp sums)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (w == 0) {
    s = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (l == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// out[r][n] = act(b[n] + sum_k W[n][k] in[r][k]) for r < R, n < N; thread
// item (n, g) takes rows g, g + G, ...  W row-major global (float4 rows).
template <int G, bool kTanh>
__device__ __forceinline__ void dense(const float* __restrict__ W, const float* __restrict__ b, int N, int K,
                                      const float* in, int ldi, float* out, int ldo, int R) {
  constexpr int RP = kRows / G;
  for (int it = threadIdx.x; it < N * G; it += kThreads) {
    const int n = it % N, g = it / N;
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
    const float4* wr = reinterpret_cast<const float4*>(W + (int64_t)n * K);
    for (int k4 = 0; k4 < K / 4; ++k4) {
      const float4 w = __ldg(wr + k4);
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(in + (g + j * G) * ldi + 4 * k4);
        acc[j] = fmaf(w.x, x.x, acc[j]);
        acc[j] = fmaf(w.y, x.y, acc[j]);
        acc[j] = fmaf(w.z, x.z, acc[j]);
        acc[j] = fmaf(w.w, x.w, acc[j]);
      }
    }
    const float bn = __ldg(b + n);
#pragma unroll
    for (int j = 0; j < RP; ++j) {
      const int r = g + j * G;
      if (r < R) out[r * ldo + n] = kTanh ? tanhf(acc[j] + bn) : acc[j] + bn;
    }
  }
}

// out[r][j] = (1 - h[r][j]^2) * sum_o d[r][o] W[o][j] (the gradient through
// y = W x and the tanh that produced h), j < J, o < N; W row-major [N][J]
template <int G>
__device__ __forceinline__ void dense_t(const float* __restrict__ W, int N, int J, const float* d, int ldd,
                                        const float* h, int ldh, float* out, int ldo, int R) {
  constexpr int RP = kRows / G;
  for (int it = threadIdx.x; it < J * G; it += kThreads) {
    const int j = it % J, g = it / J;
    float acc[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) acc[q] = 0.f;
    for (int o = 0; o < N; ++o) {
      const float w = __ldg(W + (int64_t)o * J + j);
#pragma unroll
      for (int q = 0; q < RP; ++q) acc[q] = fmaf(d[(g + q * G) * ldd + o], w, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = g + q * G;
      if (r < R) {
        const float hv = h[r * ldh + j];
        out[r * ldo + j] = acc[q] * (1.f - hv * hv);
      }
    }
  }
}

// partial gradients of y = W x + b over this CTA's rows: gW[n][k] = sum_r
// d[r][n] in[r][k] -> dst[n*K + k], gb[n] = sum_r d[r][n] -> dstb[n]
__device__ __forceinline__ void wgrad(const float* d, int ldd, const float* in, int ldi, int N, int K, int R,
                                      float* __restrict__ dst, float* __restrict__ dstb) {
  for (int e = threadIdx.x; e < N * K; e += kThreads) {
    const int n = e / K, k = e - n * K;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc = fmaf(d[r * ldd + n], in[r * ldi + k], acc);
    dst[e] = acc;
  }
  for (int n = threadIdx.x; n < N; n += kThreads) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += d[r * ldd + n];
    dstb[n] = acc;
  }
}

__host__ __device__ inline int ld_pad(int x) { return (x + 3) / 4 * 4; }

struct Smem {
  int ldx, ldz;
  int x, h1, h2, z, dz2, dz1, rows, slot, red, bytes;  // float offsets
};
__host__ __device__ inline Smem smem_layout(int K1, int NO, int S) {
  Smem s;
  s.ldx = K1;
  s.ldz = ld_pad(NO);
  s.x = 0;
  s.h1 = s.x + kRows * s.ldx;
  s.h2 = s.h1 + kRows * 2 * kH;
  s.z = s.h2 + kRows * 2 * kH;
  s.dz2 = s.z + kRows * s.ldz;
  s.dz1 = s.dz2 + kRows * 2 * kH;
  s.rows = s.dz1 + kRows * 2 * kH;  // v, dv, g_lp, g_ent per row
  s.slot = s.rows + 4 * kRows;      // [2][kRows * S]: log-prob and entropy terms
  s.red = s.slot + 2 * kRows * ld_pad(S);
  s.bytes = (s.red + 40) * 4;
  return s;
}

__global__ void __launch_bounds__(kThreads) k_ppo_grad(const Net net, const Batch bt, const Work wk, int64_t P) {
  extern __shared__ __align__(16) float su[];
  const Smem L = smem_layout(net.K1, net.NO, bt.S);
  float *x = su + L.x, *h1 = su + L.h1, *h2 = su + L.h2, *z = su + L.z, *dz2 = su + L.dz2, *dz1 = su + L.dz1;
  float *v = su + L.rows, *dv = v + kRows, *glp = dv + kRows, *gent = glp + kRows;
  float *slp = su + L.slot, *sent = slp + kRows * ld_pad(bt.S), *red = su + L.red;
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int R = (int)((bt.M - r0) < kRows ? (bt.M - r0) : kRows);
  const int S = bt.S, A = bt.A, SA = S * A, K1 = net.K1, NO = net.NO;

  // advantage normalisation over the whole minibatch (torch: a.mean(), a.std() unbiased)
  float s = 0.f;
  for (int64_t i = t; i < bt.M; i += kThreads) s += bt.scal[bt.idx[i]].z;
  const float amean = block_sum(s, red) / (float)bt.M;
  float q = 0.f;
  for (int64_t i = t; i < bt.M; i += kThreads) {
    const float d = bt.scal[bt.idx[i]].z - amean;
    q = fmaf(d, d, q);
  }
  const float astd = sqrtf(block_sum(q, red) / (float)(bt.M - 1));

  // this CTA's rows (zero-padded past obs_dim)
  for (int e = t; e < R * K1; e += kThreads) {
    const int r = e / K1, k = e - r * K1;
    x[r * L.ldx + k] = k < bt.obs_dim ? bt.obs[bt.idx[r0 + r] * bt.obs_ld + k] : 0.f;
  }
  __syncthreads();

  // forward: h1 = tanh(W1 x + b1) [actor | critic]; h2a, h2c; head z; value
  dense<2, true>(net.w[0], net.w[1], 2 * kH, K1, x, L.ldx, h1, 2 * kH, R);
  __syncthreads();
  dense<4, true>(net.w[2], net.w[3], kH, kH, h1, 2 * kH, h2, 2 * kH, R);
  dense<4, true>(net.w[6], net.w[7], kH, kH, h1 + kH, 2 * kH, h2 + kH, 2 * kH, R);
  __syncthreads();
  dense<1, false>(net.w[4], net.w[5], NO, kH, h2, 2 * kH, z, L.ldz, R);
  {  // value: one warp per row, lanes over the 64 inputs
    const int w = t >> 5, l = t & 31;
    for (int r = w; r < R; r += kThreads / 32) {
      float a = fmaf(__ldg(net.w[8] + l), h2[r * 2 * kH + kH + l], 0.f);
      a = fmaf(__ldg(net.w[8] + l + 32), h2[r * 2 * kH + kH + l + 32], a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (l == 0) v[r] = a + __ldg(net.w[9]);
    }
  }
  __syncthreads();

  // loss head (k_ppo_loss's formulas): per (row, slot) softmax statistics
  for (int it = t; it < R * S; it += kThreads) {
    const int r = it / S, sl = it - r * S;
    const float* zs = z + r * L.ldz + sl * A;
    float m = -INFINITY;
    for (int k = 0; k < A; ++k) m = fmaxf(m, zs[k]);
    float sum = 0.f, ed = 0.f;
    for (int k = 0; k < A; ++k) {
      const float d = zs[k] - m, e = __expf(d);
      sum += e;
      ed += e * d;
    }
    const float logsum = __logf(sum);
    const int a = bt.actions[bt.idx[r0 + r] * S + sl];
    slp[r * ld_pad(S) + sl] = (zs[a] - m) - logsum;
    sent[r * ld_pad(S) + sl] = logsum - ed / sum;
  }
  __syncthreads();
  // per row: the loss terms and their gradients with respect to lp, H, v
  const float inv_n = 1.f / (float)bt.M;
  float l_loss = 0.f, l_pg = 0.f, l_vf = 0.f, l_ent = 0.f;
  if (t < R) {
    float lp = 0.f, ent = 0.f;
    for (int sl = 0; sl < S; ++sl) {
      lp += slp[t * ld_pad(S) + sl];
      ent += sent[t * ld_pad(S) + sl];
    }
    const float4 sc = bt.scal[bt.idx[r0 + t]];
    const float vv = v[t];
    const float old_lp = sc.x, old_v = sc.y, an = (sc.z - amean) / (astd + 1e-8f), ret = sc.w;
    const float ratio = expf(lp - old_lp);
    const float u = ratio * an;
    const float rc = fminf(fmaxf(ratio, 1.f - bt.clip_eps), 1.f + bt.clip_eps);
    const float cc = rc * an;
    const float pg = -fminf(u, cc);
    const bool inside = ratio >= 1.f - bt.clip_eps && ratio <= 1.f + bt.clip_eps;
    const float du = u < cc ? 1.f : (u > cc ? 0.f : 0.5f), dc = 1.f - du;
    glp[t] = -(du + dc * (inside ? 1.f : 0.f)) * an * ratio * inv_n;
    gent[t] = -bt.ent_coef * inv_n;
    const float dvv = vv - old_v;
    const float dvc = fminf(fmaxf(dvv, -bt.vf_clip), bt.vf_clip);
    const float vc = old_v + dvc;
    const float e1 = (vv - ret) * (vv - ret), e2 = (vc - ret) * (vc - ret);
    const float vl = 0.5f * fmaxf(e1, e2);
    const float d1 = e1 > e2 ? 1.f : (e1 < e2 ? 0.f : 0.5f), d2 = 1.f - d1;
    const bool vin = dvv >= -bt.vf_clip && dvv <= bt.vf_clip;
    dv[t] = bt.vf_coef * inv_n * (d1 * (vv - ret) + d2 * (vc - ret) * (vin ? 1.f : 0.f));
    l_pg = pg;
    l_vf = vl;
    l_ent = ent;
    l_loss = pg + bt.vf_coef * vl - bt.ent_coef * ent;
  }
  __syncthreads();
  // d loss / d logits, in place over z (padding rows of the head: 0)
  for (int it = t; it < R * S; it += kThreads) {
    const int r = it / S, sl = it - r * S;
    float* zs = z + r * L.ldz + sl * A;
    float m = -INFINITY;
    for (int k = 0; k < A; ++k) m = fmaxf(m, zs[k]);
    float sum = 0.f, ed = 0.f;
    for (int k = 0; k < A; ++k) {
      const float d = zs[k] - m, e = __expf(d);
      sum += e;
      ed += e * d;
    }
    const float inv = 1.f / sum, logsum = __logf(sum), h = logsum - ed * inv;
    const int a = bt.actions[bt.idx[r0 + r] * S + sl];
    const float gl = glp[r], ge = gent[r];
    for (int k = 0; k < A; ++k) {
      const float d = zs[k] - m, p = __expf(d) * inv, l = d - logsum;
      zs[k] = gl * ((k == a ? 1.f : 0.f) - p) - ge * p * (l + h);
    }
  }
  for (int e = t; e < R * (NO - SA); e += kThreads) {
    const int r = e / (NO - SA);
    z[r * L.ldz + SA + (e - r * (NO - SA))] = 0.f;
  }
  __syncthreads();

  // backward: dz2 = [d h2a-pre | d h2c-pre], dz1 = d h1-pre
  dense_t<4>(net.w[4], NO, kH, z, L.ldz, h2, 2 * kH, dz2, 2 * kH, R);
  for (int e = t; e < R * kH; e += kThreads) {  // critic: d h2c = dv * wv
    const int r = e / kH, j = e - r * kH;
    const float hv = h2[r * 2 * kH + kH + j];
    dz2[r * 2 * kH + kH + j] = dv[r] * __ldg(net.w[8] + j) * (1.f - hv * hv);
  }
  __syncthreads();
  dense_t<4>(net.w[2], kH, kH, dz2, 2 * kH, h1, 2 * kH, dz1, 2 * kH, R);
  dense_t<4>(net.w[6], kH, kH, dz2 + kH, 2 * kH, h1 + kH, 2 * kH, dz1 + kH, 2 * kH, R);
  __syncthreads();

  // this CTA's partial gradients, the module's parameter order
  float* pd = wk.part + (int64_t)blockIdx.x * P;
  wgrad(dz1, 2 * kH, x, L.ldx, 2 * kH, K1, R, pd + net.off[0], pd + net.off[1]);
  wgrad(dz2, 2 * kH, h1, 2 * kH, kH, kH, R, pd + net.off[2], pd + net.off[3]);
  wgrad(z, L.ldz, h2, 2 * kH, NO, kH, R, pd + net.off[4], pd + net.off[5]);
  wgrad(dz2 + kH, 2 * kH, h1 + kH, 2 * kH, kH, kH, R, pd + net.off[6], pd + net.off[7]);
  wgrad(dv, 1, h2 + kH, 2 * kH, 1, kH, R, pd + net.off[8], pd + net.off[9]);
  // loss sums of this CTA (threads 0..R-1 hold one row each)
  const float a0 = block_sum(l_loss, red), a1 = block_sum(l_pg, red), a2 = block_sum(l_vf, red),
              a3 = block_sum(l_ent, red);
  if (t == 0) {
    float* ls = wk.lstat + 4 * blockIdx.x;
    ls[0] = a0;
    ls[1] = a1;
    ls[2] = a2;
    ls[3] = a3;
  }
}

__global__ void __launch_bounds__(kThreads) k_ppo_gsum(const Work wk, int64_t P, int nparts, int64_t M) {
  __shared__ float red[40];
  const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  float g = 0.f;
  if (p < P)
#pragma unroll 8
    for (int c = 0; c < nparts; ++c) g += wk.part[(int64_t)c * P + p];
  if (p < P) wk.grad[p] = g;
  const float s = block_sum(g * g, red);
  if (threadIdx.x == 0) wk.sq[blockIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x < 4) {
    float a = 0.f;
    for (int c = 0; c < nparts; ++c) a += wk.lstat[4 * c + threadIdx.x];
    wk.stats[threadIdx.x] = a / (float)M;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wk.step[0] += 1.f;
}

struct AdamArgs {
  float* p[kNP];
  int64_t off[kNP + 1];
  float* m;  // exp_avg [P]
  float* v;  // exp_avg_sq [P]
  const float* lr;
  float beta1, beta2, eps, max_norm;
};

__global__ void __launch_bounds__(kThreads) k_ppo_adam(const Work wk, const AdamArgs ad, int64_t P, int nsq) {
  __shared__ float red[40];
  float s = 0.f;
  for (int i = threadIdx.x; i < nsq; i += kThreads) s += wk.sq[i];
  const float norm = sqrtf(block_sum(s, red));
  const float coef = fminf(ad.max_norm / (norm + 1e-6f), 1.f);  // torch clip_grad_norm_ (clamped to 1)
  const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (p >= P) return;
  int q = 0;
  while (p >= ad.off[q + 1]) ++q;
  float* prm = ad.p[q] + (p - ad.off[q]);
  const float g = wk.grad[p] * coef;
  const float stp = wk.step[0];
  const float m = ad.beta1 * ad.m[p] + (1.f - ad.beta1) * g;
  const float v = ad.beta2 * ad.v[p] + (1.f - ad.beta2) * g * g;
  ad.m[p] = m;
  ad.v[p] = v;
  const float bc1 = 1.f - powf(ad.beta1, stp), bc2 = 1.f - powf(ad.beta2, stp);
  const float denom = sqrtf(v) / sqrtf(bc2) + ad.eps;
  *prm -= (*ad.lr / bc1) * m / denom;
}

}  // namespace vyu

extern "C" {

int vy_ppo_update_workspace(int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M, int64_t out[4]) {
  if (hidden != vyu::kH || obs_dim < 1 || S < 1 || A < 2 || M < 2) return VY_ERR_UNSUPPORTED;
  const int K1 = (obs_dim + 7) / 8 * 8, NO = (S * A + 7) / 8 * 8;
  const int64_t P = (int64_t)2 * vyu::kH * K1 + 2 * vyu::kH + vyu::kH * vyu::kH + vyu::kH + (int64_t)NO * vyu::kH + NO +
                    vyu::kH * vyu::kH + vyu::kH + vyu::kH + 1;
  const int64_t grid = (M + vyu::kRows - 1) / vyu::kRows;
  const int64_t nsq = (P + vyu::kThreads - 1) / vyu::kThreads;
  out[0] = P;                                // parameters
  out[1] = grid * P + grid * 4 + nsq;       // float workspace: partials, loss partials, block squares
  out[2] = grid;                             // k_ppo_grad CTAs
  out[3] = vyu::smem_layout(K1, NO, S).bytes;
  return out[3] > 227 * 1024 ? VY_ERR_UNSUPPORTED : VY_OK;
}

int vy_ppo_update_grad(const float* const* weights, int32_t obs_dim, int32_t S, int32_t A, int32_t hidden,
                       const float* obs, int64_t obs_ld, const uint8_t* actions, const float* scal4,
                       const int64_t* idx, int64_t M, float clip_eps, float vf_clip, float vf_coef, float ent_coef,
                       float* work, float* grad_out, float* stats, float* step, void* stream) {
  int64_t ws[4];
  if (int rc = vy_ppo_update_workspace(obs_dim, S, A, hidden, M, ws)) return rc;
  if (!weights || !obs || !actions || !scal4 || !idx || !work || !grad_out || !stats || !step) return VY_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(scal4) & 15u) != 0) return VY_ERR_ARG;
  vyu::Net net{};
  const int K1 = (obs_dim + 7) / 8 * 8, NO = (S * A + 7) / 8 * 8, H = vyu::kH;
  const int64_t sizes[vyu::kNP] = {2 * H * K1, 2 * H, H * H, H, (int64_t)NO * H, NO, H * H, H, H, 1};
  net.off[0] = 0;
  for (int i = 0; i < vyu::kNP; ++i) {
    if (!weights[i] || (reinterpret_cast<uintptr_t>(weights[i]) & 15u) != 0) return VY_ERR_ARG;
    net.w[i] = weights[i];
    net.off[i + 1] = net.off[i] + sizes[i];
  }
  net.K1 = K1;
  net.NO = NO;
  const int64_t P = ws[0], grid = ws[2];
  vyu::Batch bt{obs, obs_ld, obs_dim, actions, reinterpret_cast<const float4*>(scal4), idx, M, S, A,
                clip_eps, vf_clip, vf_coef, ent_coef};
  vyu::Work wk{work, work + grid * P, grad_out, work + grid * P + grid * 4, stats, step};
  const int smem = (int)ws[3];
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(vyu::k_ppo_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return VY_ERR_CUDA;
    attr = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  vyu::k_ppo_grad<<<(unsigned)grid, vyu::kThreads, smem, st>>>(net, bt, wk, P);
  const unsigned nsq = (unsigned)((P + vyu::kThreads - 1) / vyu::kThreads);
  vyu::k_ppo_gsum<<<nsq, vyu::kThreads, 0, st>>>(wk, P, (int)grid, M);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

int vy_ppo_update_adam(float* const* params, int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M,
                       float* work, const float* grad, float* exp_avg, float* exp_avg_sq, const float* lr,
                       const float* step, float beta1, float beta2, float eps, float max_grad_norm, void* stream) {
  int64_t ws[4];
  if (int rc = vy_ppo_update_workspace(obs_dim, S, A, hidden, M, ws)) return rc;
  if (!params || !work || !grad || !exp_avg || !exp_avg_sq || !lr || !step) return VY_ERR_ARG;
  const int K1 = (obs_dim + 7) / 8 * 8, NO = (S * A + 7) / 8 * 8, H = vyu::kH;
  const int64_t sizes[vyu::kNP] = {2 * H * K1, 2 * H, H * H, H, (int64_t)NO * H, NO, H * H, H, H, 1};
  vyu::AdamArgs ad{};
  ad.off[0] = 0;
  for (int i = 0; i < vyu::kNP; ++i) {
    if (!params[i]) return VY_ERR_ARG;
    ad.p[i] = params[i];
    ad.off[i + 1] = ad.off[i] + sizes[i];
  }
  ad.m = exp_avg;
  ad.v = exp_avg_sq;
  ad.lr = lr;
  ad.beta1 = beta1;
  ad.beta2 = beta2;
  ad.eps = eps;
  ad.max_norm = max_grad_norm;
  const int64_t P = ws[0], grid = ws[2];
  vyu::Work wk{work, work + grid * P, const_cast<float*>(grad), work + grid * P + grid * 4, nullptr,
               const_cast<float*>(step)};
  const unsigned nsq = (unsigned)((P + vyu::kThreads - 1) / vyu::kThreads);
  vyu::k_ppo_adam<<<nsq, vyu::kThreads, 0, (cudaStream_t)stream>>>(wk, ad, P, (int)nsq);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

}  // extern "C"
