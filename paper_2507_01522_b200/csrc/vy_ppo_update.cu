// vy_ppo_update.cu — one PPO minibatch update (forward, clipped loss,
// backward, global-norm clipping, Adam) in three kernel launches, for the
// small batches the paper trains on (PPO(16): 1200-sample minibatches).
//
// The autograd path (ppo.py _update_body) is ~70 launches per minibatch —
// weight casts, three GEMM pairs, bias column sums, tanh forward/backward,
// the loss kernel, the norm, Adam — each a few microseconds of latency on an
// idle GPU at these sizes (~190 us per minibatch, CUDA graph replayed).  Here:
//   k_ppo_grad  (ceil(M/8) CTAs x 512 threads): every CTA normalises the
//     minibatch's advantages (mean / unbiased std over all M rows, the same
//     fixed-order reduction in every CTA), gathers its <= 8 rows, runs the
//     actor-critic forward in fp32 from transposed copies of the live fp32
//     weight matrices (L2-resident; k_ppo_adam keeps them in step), 
//     the loss head of k_ppo_loss (same formulas: log-softmax per slot,
//     entropy, clipped surrogate, clipped value loss), the backward through
//     the three layers, and writes its partial weight gradient (sum over its
//     rows) and loss sums;
//   k_ppo_gsum  (four threads per parameter): the partials summed over the
//     CTAs in a fixed order (contiguous quarters, then the quarters in order) -> the flat gradient; per-block sums of
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

#ifdef VY_PPO_PROF  // phase timing build (scripts/probe_ppo_phases.py): clock64 deltas of CTA 0 thread 0
__device__ unsigned long long g_upd_prof[16];
#define UPD_MARK(i)                                   \
  if (blockIdx.x == 0 && threadIdx.x == 0) {          \
    const unsigned long long now_ = clock64();        \
    g_upd_prof[i] += now_ - prof_last;                \
    prof_last = now_;                                 \
  }
#else
#define UPD_MARK(i)
#endif

// rows per CTA: 8, or 16 when 8 would need more than one wave of CTAs
// rows per CTA: the fewest of 8 / 10 / 16 that keep the grid to one wave
// (PPO(16)'s 1200-row minibatches: 10 rows, 120 CTAs)
__host__ __device__ inline int rows_per_cta(int64_t M, int num_sms) {
  return M <= 8LL * num_sms ? 8 : (M <= 10LL * num_sms ? 10 : 16);
}
// row groups per output for the layer shapes (rows per thread = ROWS / G)
__host__ __device__ constexpr int g_l1(int rows) { return rows == 10 ? 2 : 4; }    // 128 outputs
__host__ __device__ constexpr int g_64(int rows) { return rows == 10 ? 5 : 8; }    // 64 outputs
__host__ __device__ constexpr int g_head(int rows) { return rows >= 16 ? 2 : 1; }  // ~360 outputs
constexpr int kThreads = 512;
constexpr int kH = 64;         // hidden width per branch
constexpr int kNP = 10;        // parameter tensors (ActorCritic order)

struct Net {
  const float* w[kNP];  // w1, b1, wa2, ba2, wh, bh, wc2, bc2, wv, bv
  const float* wt;      // W1 transposed [K1][2H] (coalesced first-layer reads)
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
  const float* adv_stats;  // {mean, std} of the minibatch's advantages, or null (computed here)
  int64_t M;
  int S, A;
  float clip_eps, vf_clip, vf_coef, ent_coef;
};

struct Work {
  int64_t pld;   // row stride of the partials (P rounded up to 4: 16-byte aligned rows)
  float* part;   // [grid][pld] per-CTA gradient partials
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

// out[r][n] = act(b[n] + sum_k WT[k][n] in[r][k]) for r < R, n < N; thread
// item (n, g) takes rows g, g + G, ...  WT: the transposed weight [K][N] in
// global memory (the threads of a warp read consecutive n: coalesced).
template <int ROWS, int G, bool kTanh>
__device__ __forceinline__ void dense_gt(const float* __restrict__ WT, const float* __restrict__ b, int N, int K,
                                         const float* in, int ldi, float* out, int ldo, int R) {
  static_assert(ROWS % G == 0, "row groups must divide the rows");
  constexpr int RP = ROWS / G;
  for (int it = threadIdx.x; it < N * G; it += kThreads) {
    const int n = it % N, g = it / N;
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < K; k += 4) {
      const float w0 = __ldg(WT + (int64_t)k * N + n), w1 = __ldg(WT + (int64_t)(k + 1) * N + n);
      const float w2 = __ldg(WT + (int64_t)(k + 2) * N + n), w3 = __ldg(WT + (int64_t)(k + 3) * N + n);
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(in + (g + j * G) * ldi + k);
        acc[j] = fmaf(w0, x.x, acc[j]);
        acc[j] = fmaf(w1, x.y, acc[j]);
        acc[j] = fmaf(w2, x.z, acc[j]);
        acc[j] = fmaf(w3, x.w, acc[j]);
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

// the same from a row-major weight staged in shared memory, row stride ldw
// (kH + 4: 16-byte row reads by consecutive n fall in distinct banks)
template <int ROWS, int G, bool kTanh>
__device__ __forceinline__ void dense_s(const float* W, int ldw, const float* __restrict__ b, int N, int K,
                                        const float* in, int ldi, float* out, int ldo, int R) {
  static_assert(ROWS % G == 0, "row groups must divide the rows");
  constexpr int RP = ROWS / G;
  for (int it = threadIdx.x; it < N * G; it += kThreads) {
    const int n = it % N, g = it / N;
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < K; k += 4) {
      const float4 w = *reinterpret_cast<const float4*>(W + n * ldw + k);
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(in + (g + j * G) * ldi + k);
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
// y = W x and the tanh that produced h), j < J, o < N; W row-major in shared
// memory (row stride ldw; consecutive j: conflict-free), N a multiple of 4
template <int ROWS, int G>
__device__ __forceinline__ void dense_t(const float* W, int ldw, int N, int J, const float* d, int ldd,
                                        const float* h, int ldh, float* out, int ldo) {
  static_assert(ROWS % G == 0, "row groups must divide the rows");
  constexpr int RP = ROWS / G;
  for (int it = threadIdx.x; it < J * G; it += kThreads) {
    const int j = it % J, g = it / J;
    float acc[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) acc[q] = 0.f;
#pragma unroll 4
    for (int o = 0; o < N; o += 4) {
      const float w0 = W[o * ldw + j], w1 = W[(o + 1) * ldw + j], w2 = W[(o + 2) * ldw + j],
                  w3 = W[(o + 3) * ldw + j];
#pragma unroll
      for (int q = 0; q < RP; ++q) {
        const float4 dq = *reinterpret_cast<const float4*>(d + (g + q * G) * ldd + o);
        acc[q] = fmaf(dq.x, w0, acc[q]);
        acc[q] = fmaf(dq.y, w1, acc[q]);
        acc[q] = fmaf(dq.z, w2, acc[q]);
        acc[q] = fmaf(dq.w, w3, acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = g + q * G;
      const float hv = h[r * ldh + j];
      out[r * ldo + j] = acc[q] * (1.f - hv * hv);
    }
  }
}

// partial gradients of y = W x + b over this CTA's rows, register-tiled:
// gW[n][k] = sum_r d[r][n] in[r][k] -> dst[n*K + k], gb[n] = sum_r d[r][n].
// A warp owns a 32 (n) x 16 (k) block, a lane a 4 x 4 tile (lanes 4i..4i+3:
// n-quad i, k-quads 0..3), so per row a warp reads 8 d-quads and 4 in-quads
// (one wavefront each) for 16 FMAs per lane.  N, K, ldd, ldi multiples of 4,
// dst rows 16-byte aligned; d is zero past the CTA's rows.
template <int ROWS>
__device__ __forceinline__ void wgrad(const float* d, int ldd, const float* in, int ldi, int N, int K,
                                      float* __restrict__ dst, float* __restrict__ dstb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NB = (N + 31) / 32, KB = (K + 15) / 16;
  for (int wb = warp; wb < NB * KB; wb += kThreads / 32) {
    const int bn = wb / KB, bk = wb - bn * KB;
    const int n = bn * 32 + (lane >> 2) * 4, k = bk * 16 + (lane & 3) * 4;
    if (n < N && k < K) {
      float4 acc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const float4 dq = *reinterpret_cast<const float4*>(d + r * ldd + n);
        const float4 xq = *reinterpret_cast<const float4*>(in + r * ldi + k);
        const float dd[4] = {dq.x, dq.y, dq.z, dq.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i].x = fmaf(dd[i], xq.x, acc[i].x);
          acc[i].y = fmaf(dd[i], xq.y, acc[i].y);
          acc[i].z = fmaf(dd[i], xq.z, acc[i].z);
          acc[i].w = fmaf(dd[i], xq.w, acc[i].w);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) *reinterpret_cast<float4*>(dst + (int64_t)(n + i) * K + k) = acc[i];
    }
  }
  for (int n = threadIdx.x; n < N; n += kThreads) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc += d[r * ldd + n];
    dstb[n] = acc;
  }
}

// the same with one thread per 4 k (any N, ldd; the value head): gW[n][k] = sum_r
// d[r][n] in[r][k] -> dst[n*K + k], gb[n] = sum_r d[r][n] -> dstb[n].  All
// ROWS rows (d is zero past the CTA's rows), four k per thread: 16-byte
// loads, the whole row loop unrolled so its loads are in flight together.
template <int ROWS>
__device__ __forceinline__ void wgrad_rows(const float* d, int ldd, const float* in, int ldi, int N, int K,
                                      float* __restrict__ dst, float* __restrict__ dstb) {
  const int K4 = K / 4;
  for (int e = threadIdx.x; e < N * K4; e += kThreads) {
    const int n = e / K4, k4 = e - n * K4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const float dn = d[r * ldd + n];
      const float4 x = *reinterpret_cast<const float4*>(in + r * ldi + 4 * k4);
      acc.x = fmaf(dn, x.x, acc.x);
      acc.y = fmaf(dn, x.y, acc.y);
      acc.z = fmaf(dn, x.z, acc.z);
      acc.w = fmaf(dn, x.w, acc.w);
    }
    float* o = dst + (int64_t)n * K + 4 * k4;  // dst offsets are not 16-byte aligned in general
    o[0] = acc.x;
    o[1] = acc.y;
    o[2] = acc.z;
    o[3] = acc.w;
  }
  for (int n = threadIdx.x; n < N; n += kThreads) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc += d[r * ldd + n];
    dstb[n] = acc;
  }
}

// mean and unbiased standard deviation of scal[idx[i]].z, i < M (fixed-order block reductions)
__device__ __forceinline__ void adv_mean_std(const float4* __restrict__ scal, const int64_t* __restrict__ idx,
                                             int64_t M, float* red, float& mean, float& std) {
  float s = 0.f;
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) s += scal[idx[i]].z;
  mean = block_sum(s, red) / (float)M;
  float q = 0.f;
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    const float d = scal[idx[i]].z - mean;
    q = fmaf(d, d, q);
  }
  std = sqrtf(block_sum(q, red) / (float)(M - 1));
}

// the advantage statistics of every minibatch of an update: block b = epoch
// b / nmb, minibatch b % nmb (rows perms[epoch][k*mb .. (k+1)*mb))
__global__ void __launch_bounds__(kThreads) k_adv_stats(const float4* __restrict__ scal,
                                                         const int64_t* __restrict__ perms, int64_t n, int nmb,
                                                         int64_t mb, float* __restrict__ out) {
  __shared__ float red[40];
  const int e = blockIdx.x / nmb, k = blockIdx.x - e * nmb;
  float mean, std;
  adv_mean_std(scal, perms + (int64_t)e * n + (int64_t)k * mb, mb, red, mean, std);
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = mean;
    out[2 * blockIdx.x + 1] = std;
  }
}

__host__ __device__ inline int ld_pad(int x) { return (x + 3) / 4 * 4; }
constexpr int kLdw = kH + 4;  // row stride of the staged [*][kH] weights

struct Smem {
  int ldx, ldz;
  int wa2, wc2, wh;                                    // staged weights (row stride kLdw)
  int x, h1, h2, z, dz2, dz1, rows, slot, red, bytes;  // float offsets
};
__host__ __device__ inline Smem smem_layout(int rows, int K1, int NO, int S) {
  Smem s;
  s.ldx = K1;
  s.ldz = ld_pad(NO);
  s.wa2 = 0;
  s.wc2 = s.wa2 + kH * kLdw;
  s.wh = s.wc2 + kH * kLdw;
  s.x = s.wh + NO * kLdw;
  s.h1 = s.x + rows * s.ldx;
  s.h2 = s.h1 + rows * 2 * kH;
  s.z = s.h2 + rows * 2 * kH;
  s.dz2 = s.z + rows * s.ldz;
  s.dz1 = s.dz2 + rows * 2 * kH;
  s.rows = s.dz1 + rows * 2 * kH;  // v, dv, g_lp, g_ent per row
  s.slot = s.rows + 4 * rows;      // [2][rows * S]: log-prob and entropy terms
  s.red = s.slot + 2 * rows * ld_pad(S);
  s.bytes = (s.red + 40) * 4;
  return s;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
}

// [n][kH] row-major weight -> shared rows of stride kLdw, 16-byte async copies
__device__ __forceinline__ void stage_weight(float* dst, const float* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n * (kH / 4); i += kThreads) {
    const int r = i / (kH / 4), c = i - r * (kH / 4);
    cp_async16(dst + r * kLdw + 4 * c, src + (int64_t)r * kH + 4 * c);
  }
}

template <int ROWS>
__global__ void __launch_bounds__(kThreads, 1) k_ppo_grad(const Net net, const Batch bt, const Work wk, int64_t P) {
  extern __shared__ __align__(16) float su[];
  const Smem L = smem_layout(ROWS, net.K1, net.NO, bt.S);
  float *x = su + L.x, *h1 = su + L.h1, *h2 = su + L.h2, *z = su + L.z, *dz2 = su + L.dz2, *dz1 = su + L.dz1;
  float *v = su + L.rows, *dv = v + ROWS, *glp = dv + ROWS, *gent = glp + ROWS;
  float *slp = su + L.slot, *sent = slp + ROWS * ld_pad(bt.S), *red = su + L.red;
  float *swa2 = su + L.wa2, *swc2 = su + L.wc2, *swh = su + L.wh;
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int R = (int)((bt.M - r0) < ROWS ? (bt.M - r0) : ROWS);
  const int S = bt.S, A = bt.A, SA = S * A, K1 = net.K1, NO = net.NO;
#ifdef VY_PPO_PROF
  unsigned long long prof_last = clock64();
#endif

  // the second layers and the head into shared memory, in flight during the
  // advantage statistics, the row gather and the first layer
  stage_weight(swa2, net.w[2], kH);
  stage_weight(swc2, net.w[6], kH);
  stage_weight(swh, net.w[4], NO);
  asm volatile("cp.async.commit_group;" ::: "memory");

  // advantage normalisation over the whole minibatch (torch: a.mean(), a.std()
  // unbiased): precomputed for the update's minibatches (vy_ppo_adv_stats), or here
  float amean, astd;
  if (bt.adv_stats) {
    amean = bt.adv_stats[0];
    astd = bt.adv_stats[1];
  } else {
    adv_mean_std(bt.scal, bt.idx, bt.M, red, amean, astd);
  }

  // this CTA's rows (zero-padded past obs_dim)
  for (int e = t; e < ROWS * K1; e += kThreads) {  // rows past R: zeros (finite activations, zero gradients)
    const int r = e / K1, k = e - r * K1;
    x[r * L.ldx + k] = (r < R && k < bt.obs_dim) ? bt.obs[bt.idx[r0 + r] * bt.obs_ld + k] : 0.f;
  }
  __syncthreads();
  UPD_MARK(0);

  // forward: h1 = tanh(W1 x + b1) [actor | critic]; h2a, h2c; head z; value
  dense_gt<ROWS, g_l1(ROWS), true>(net.wt, net.w[1], 2 * kH, K1, x, L.ldx, h1, 2 * kH, ROWS);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  UPD_MARK(1);
  dense_s<ROWS, g_64(ROWS), true>(swa2, kLdw, net.w[3], kH, kH, h1, 2 * kH, h2, 2 * kH, ROWS);
  dense_s<ROWS, g_64(ROWS), true>(swc2, kLdw, net.w[7], kH, kH, h1 + kH, 2 * kH, h2 + kH, 2 * kH, ROWS);
  __syncthreads();
  dense_s<ROWS, g_head(ROWS), false>(swh, kLdw, net.w[5], NO, kH, h2, 2 * kH, z, L.ldz, R);
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

  UPD_MARK(2);
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
  for (int e = t; e < (ROWS - R) * L.ldz; e += kThreads) z[R * L.ldz + e] = 0.f;  // rows past R: no gradient
  if (t >= R && t < ROWS) dv[t] = 0.f;
  __syncthreads();

  UPD_MARK(3);
  // backward: dz2 = [d h2a-pre | d h2c-pre], dz1 = d h1-pre
  dense_t<ROWS, g_64(ROWS)>(swh, kLdw, NO, kH, z, L.ldz, h2, 2 * kH, dz2, 2 * kH);
  for (int e = t; e < ROWS * kH; e += kThreads) {  // critic: d h2c = dv * wv
    const int r = e / kH, j = e - r * kH;
    const float hv = h2[r * 2 * kH + kH + j];
    dz2[r * 2 * kH + kH + j] = dv[r] * __ldg(net.w[8] + j) * (1.f - hv * hv);
  }
  __syncthreads();
  dense_t<ROWS, g_64(ROWS)>(swa2, kLdw, kH, kH, dz2, 2 * kH, h1, 2 * kH, dz1, 2 * kH);
  dense_t<ROWS, g_64(ROWS)>(swc2, kLdw, kH, kH, dz2 + kH, 2 * kH, h1 + kH, 2 * kH, dz1 + kH, 2 * kH);
  __syncthreads();

  UPD_MARK(4);
  // this CTA's partial gradients, the module's parameter order
  float* pd = wk.part + (int64_t)blockIdx.x * wk.pld;
  wgrad<ROWS>(dz1, 2 * kH, x, L.ldx, 2 * kH, K1, pd + net.off[0], pd + net.off[1]);
  wgrad<ROWS>(dz2, 2 * kH, h1, 2 * kH, kH, kH, pd + net.off[2], pd + net.off[3]);
  wgrad<ROWS>(z, L.ldz, h2, 2 * kH, NO, kH, pd + net.off[4], pd + net.off[5]);
  wgrad<ROWS>(dz2 + kH, 2 * kH, h1 + kH, 2 * kH, kH, kH, pd + net.off[6], pd + net.off[7]);
  wgrad_rows<ROWS>(dv, 1, h2 + kH, 2 * kH, 1, kH, pd + net.off[8], pd + net.off[9]);
  // loss sums of this CTA (threads 0..R-1 hold one row each)
  UPD_MARK(5);
  if (t < 32) {  // rows live on threads 0..ROWS-1 (warp 0): one warp reduction of the four sums
    float a[4] = {l_loss, l_pg, l_vf, l_ent};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[i] += __shfl_down_sync(0xffffffffu, a[i], o);
    if (t == 0) {
      float* ls = wk.lstat + 4 * blockIdx.x;
      ls[0] = a[0];
      ls[1] = a[1];
      ls[2] = a[2];
      ls[3] = a[3];
    }
  }
}

constexpr int kSumThreads = 256;
constexpr int kSplit = 4;  // threads per parameter in k_ppo_gsum

// four consecutive threads per parameter sum contiguous quarters of the CTA
// partials; the quarter sums are added in quarter order (deterministic)
__global__ void __launch_bounds__(kSumThreads) k_ppo_gsum(const Work wk, int64_t P, int nparts, int64_t M) {
  __shared__ float red[40];
  const int64_t p = ((int64_t)blockIdx.x * kSumThreads + threadIdx.x) / kSplit;
  const int qtr = threadIdx.x % kSplit;
  const int per = (nparts + kSplit - 1) / kSplit, c0 = qtr * per, c1 = min(nparts, c0 + per);
  float g = 0.f;
  if (p < P)
#pragma unroll 8
    for (int c = c0; c < c1; ++c) g += wk.part[(int64_t)c * wk.pld + p];
  // in-order combine of the kSplit range sums (lanes base .. base + kSplit - 1 of one warp)
  static_assert(kSplit >= 1 && kSplit <= 32 && (kSplit & (kSplit - 1)) == 0, "kSplit: a power of two <= 32");
  const unsigned FULL = 0xffffffffu;
  const int base = (threadIdx.x & 31) & ~(kSplit - 1);
  float tot = __shfl_sync(FULL, g, base);
#pragma unroll
  for (int i = 1; i < kSplit; ++i) tot += __shfl_sync(FULL, g, base + i);
  g = tot;
  const bool lead = qtr == 0 && p < P;
  if (lead) wk.grad[p] = g;
  const float s = block_sum(lead ? g * g : 0.f, red);
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
  float* w1t;  // W1 transposed, kept in step with W1
  int K1;
  int64_t off[kNP + 1];
  float* m;  // exp_avg [P]
  float* v;  // exp_avg_sq [P]
  const float* lr;
  float beta1, beta2, eps, max_norm;
};

__global__ void __launch_bounds__(kSumThreads) k_ppo_adam(const Work wk, const AdamArgs ad, int64_t P, int nsq) {
  __shared__ float red[40];
  float s = 0.f;
  for (int i = threadIdx.x; i < nsq; i += kSumThreads) s += wk.sq[i];
  const float norm = sqrtf(block_sum(s, red));
  const float coef = fminf(ad.max_norm / (norm + 1e-6f), 1.f);  // torch clip_grad_norm_ (clamped to 1)
  const int64_t p = (int64_t)blockIdx.x * kSumThreads + threadIdx.x;
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
  const float np = *prm - (*ad.lr / bc1) * m / denom;
  *prm = np;
  if (q == 0) {  // W1 element (row, col) of [2H][K1] -> [col][row] of the copy
    const int64_t row = p / ad.K1, col = p - row * ad.K1;
    ad.w1t[col * (2 * kH) + row] = np;
  }
}

}  // namespace vyu

namespace {
int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
  }
  return n;
}
struct Geo {
  int K1, NO, rows;
  int64_t P, pld, grid, nsq, sizes[vyu::kNP];
};
int geo(int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M, Geo& g) {
  if (hidden != vyu::kH || obs_dim < 1 || S < 1 || A < 2 || M < 2) return VY_ERR_UNSUPPORTED;
  const int H = vyu::kH;
  g.K1 = (obs_dim + 7) / 8 * 8;
  g.NO = (S * A + 7) / 8 * 8;
  const int64_t sizes[vyu::kNP] = {2 * H * g.K1, 2 * H, H * H, H, (int64_t)g.NO * H, g.NO, H * H, H, H, 1};
  g.P = 0;
  for (int i = 0; i < vyu::kNP; ++i) g.sizes[i] = sizes[i], g.P += sizes[i];
  g.pld = (g.P + 3) / 4 * 4;
  g.rows = vyu::rows_per_cta(M, num_sms());
  g.grid = (M + g.rows - 1) / g.rows;
  g.nsq = (g.P * vyu::kSplit + vyu::kSumThreads - 1) / vyu::kSumThreads;  // k_ppo_gsum blocks
  return vyu::smem_layout(g.rows, g.K1, g.NO, S).bytes > 227 * 1024 ? VY_ERR_UNSUPPORTED : VY_OK;
}
}  // namespace

extern "C" {

int vy_ppo_update_workspace(int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M, int64_t out[4]) {
  Geo g;
  if (int rc = geo(obs_dim, S, A, hidden, M, g)) return rc;
  out[0] = g.P;                                // parameters
  out[1] = g.grid * g.pld + g.grid * 4 + g.nsq;  // float workspace: partials, loss partials, block squares
  out[2] = g.grid;                             // k_ppo_grad CTAs
  out[3] = vyu::smem_layout(g.rows, g.K1, g.NO, S).bytes;
  return VY_OK;
}

int vy_ppo_update_grad(const float* const* weights, const float* w1t, int32_t obs_dim, int32_t S, int32_t A,
                       int32_t hidden, const float* obs, int64_t obs_ld, const uint8_t* actions, const float* scal4,
                       const int64_t* idx, const float* adv_stats, int64_t M, float clip_eps, float vf_clip, float vf_coef, float ent_coef,
                       float* work, float* grad_out, float* stats, float* step, void* stream) {
  Geo g;
  if (int rc = geo(obs_dim, S, A, hidden, M, g)) return rc;
  if (!weights || !w1t || !obs || !actions || !scal4 || !idx || !work || !grad_out || !stats || !step)
    return VY_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(scal4) & 15u) != 0) return VY_ERR_ARG;
  vyu::Net net{};
  net.off[0] = 0;
  for (int i = 0; i < vyu::kNP; ++i) {
    if (!weights[i] || (reinterpret_cast<uintptr_t>(weights[i]) & 15u) != 0) return VY_ERR_ARG;
    net.w[i] = weights[i];
    net.off[i + 1] = net.off[i] + g.sizes[i];
  }
  net.wt = w1t;
  net.K1 = g.K1;
  net.NO = g.NO;
  const int64_t P = g.P, grid = g.grid;
  vyu::Batch bt{obs, obs_ld, obs_dim, actions, reinterpret_cast<const float4*>(scal4), idx, adv_stats, M, S, A,
                clip_eps, vf_clip, vf_coef, ent_coef};
  const int64_t pld = g.pld;
  if ((reinterpret_cast<uintptr_t>(work) & 15u) != 0) return VY_ERR_ARG;
  vyu::Work wk{pld, work, work + grid * pld, grad_out, work + grid * pld + grid * 4, stats, step};
  const int smem = vyu::smem_layout(g.rows, g.K1, g.NO, S).bytes;
  auto* kern = g.rows == 8 ? vyu::k_ppo_grad<8> : g.rows == 10 ? vyu::k_ppo_grad<10> : vyu::k_ppo_grad<16>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return VY_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  kern<<<(unsigned)grid, vyu::kThreads, smem, st>>>(net, bt, wk, P);
  vyu::k_ppo_gsum<<<(unsigned)g.nsq, vyu::kSumThreads, 0, st>>>(wk, P, (int)grid, M);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

int vy_ppo_update_adam(float* const* params, float* w1t, int32_t obs_dim, int32_t S, int32_t A, int32_t hidden,
                       int64_t M, float* work, const float* grad, float* exp_avg, float* exp_avg_sq, const float* lr,
                       const float* step, float beta1, float beta2, float eps, float max_grad_norm, void* stream) {
  Geo g;
  if (int rc = geo(obs_dim, S, A, hidden, M, g)) return rc;
  if (!params || !w1t || !work || !grad || !exp_avg || !exp_avg_sq || !lr || !step) return VY_ERR_ARG;
  vyu::AdamArgs ad{};
  ad.off[0] = 0;
  for (int i = 0; i < vyu::kNP; ++i) {
    if (!params[i]) return VY_ERR_ARG;
    ad.p[i] = params[i];
    ad.off[i + 1] = ad.off[i] + g.sizes[i];
  }
  ad.w1t = w1t;
  ad.K1 = g.K1;
  ad.m = exp_avg;
  ad.v = exp_avg_sq;
  ad.lr = lr;
  ad.beta1 = beta1;
  ad.beta2 = beta2;
  ad.eps = eps;
  ad.max_norm = max_grad_norm;
  const int64_t P = g.P, grid = g.grid;
  vyu::Work wk{g.pld, work, work + grid * g.pld, const_cast<float*>(grad), work + grid * g.pld + grid * 4, nullptr,
               const_cast<float*>(step)};
  const unsigned nadam = (unsigned)((P + vyu::kSumThreads - 1) / vyu::kSumThreads);
  vyu::k_ppo_adam<<<nadam, vyu::kSumThreads, 0, (cudaStream_t)stream>>>(wk, ad, P, (int)g.nsq);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

#ifdef VY_PPO_PROF
int vy_upd_prof_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vyu::g_upd_prof, sizeof(vyu::g_upd_prof)) == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}
#endif

int vy_ppo_adv_stats(const float* scal4, const int64_t* perms, int64_t n, int32_t count, int32_t nmb, int64_t mb,
                     float* out, void* stream) {
  if (!scal4 || !perms || !out || n < 2 || count < 1 || nmb < 1 || mb < 2 || (int64_t)nmb * mb > n ||
      (reinterpret_cast<uintptr_t>(scal4) & 15u) != 0)
    return VY_ERR_ARG;
  vyu::k_adv_stats<<<(unsigned)(count * nmb), vyu::kThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(scal4), perms, n, nmb, mb, out);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

}  // extern "C"
