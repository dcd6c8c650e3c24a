// vy_policy.cu — the PPO rollout's policy forward on the 5th-generation
// tensor cores: one persistent sm_100a kernel per rollout step that reads the
// float32 observations the env step just wrote and writes the sampled
// multi-discrete actions, their log-probability and the value estimate.
//
// Network (ppo.py ActorCritic, PureJaxRL's default actor-critic, PAPER.md
// 465-490): h1 = tanh(W1 x + b1) for actor and critic at once ([2H x K1],
// rows 0..H-1 actor, H..2H-1 critic), h2a = tanh(Wa2 h1a + b2a),
// h2c = tanh(Wc2 h1c + b2c), logits = Wh h2a + bh (S slots x A actions),
// value = wv . h2c + bv.  Numerics follow the bf16 autocast forward the
// unfused path runs (cuBLAS bf16 GEMMs with fp32 accumulation, bf16 outputs,
// bf16 tanh): every layer output is rounded to bf16 before the next use.
//
// Per 32-row sub-tile (one CTA per SM, 17 warps, persistent over sub-tiles;
// the rows are replicated 4x into the M = 128 MMA tile, see k_policy_step):
//   obs rows (32 x obs_ld float32, one contiguous block) -> shared
//     memory with one bulk async copy (TMA engine, mbarrier completion), the
//     next tile's copy in flight while this tile computes;
//   convert to bf16 in the UMMA K-major no-swizzle layout ([k/8][row][8]);
//   layer 1: 7 x tcgen05.mma (M=128, N=2H=128, K=16) into TMEM columns 0..127;
//   epilogue 1: tcgen05.ld -> bias, tanh (SFU), bf16 -> shared A operand;
//   layer 2: actor and critic halves, 2 x 4 tcgen05.mma (N=64) -> TMEM 128..255;
//   epilogue 2: actor -> shared A operand, critic -> value dot product;
//   layer 3: head, 2 tcgen05.mma chains (N=256 + N=160; slot s in columns
//     24s..24s+A-1) -> TMEM 0..415;
//   epilogue 3: per (row, slot): bf16 logits, max / exp / sum, one uniform
//     from the in-kernel counter-based stream, inverse-CDF categorical sample,
//     log-probability; per-row sums through shared memory.
// Weights (~94 KB bf16, pre-laid-out by the host in the UMMA layout) are
// bulk-copied into shared memory once per CTA.  One thread issues every MMA
// and commits to an mbarrier the epilogue warps wait on.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/voltyard_b200.h"

#include "vy_umma.cuh"

namespace vyp {

// Rows are processed 32 at a time (a sub-tile), each replicated into the four
// 32-row quarters of the M = 128 MMA tile: every TMEM lane quadrant then holds
// all 32 rows, so warp w (which may only read lane quadrant w % 4) can take
// any column range of any row.  Epilogues 1 and 2: warp w < 16 owns 8-column
// chunk w; the head: warp w owns slot w (S <= 17 warps).  The MMAs compute 4x
// the rows they need — the tensor cores are idle here anyway — and a 4096-row
// rollout step spreads over 128 CTAs instead of 32.
__global__ void __launch_bounds__(kThreads, 1)
    k_policy_step(const float* __restrict__ obs, int64_t N, Geo G, const uint8_t* __restrict__ wpack,
                  const float* __restrict__ fpack, uint64_t seed, unsigned long long* counter,
                  uint8_t* __restrict__ actions, float* __restrict__ logp, float* __restrict__ value,
                  float* __restrict__ logits_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tq = (uint32_t)(32 * (warp & 3)) << 16;  // this warp's TMEM lane quadrant
  const uint32_t s_base = smem_u32(sm);
  const uint32_t bar_w = s_base + G.off_bar, bar_obs = bar_w + 8, bar_mma = bar_w + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + G.off_bar + 24);
  float* fp = reinterpret_cast<float*>(sm + G.off_f);
  const float *b1 = fp, *b2a = fp + 2 * kH, *b2c = fp + 3 * kH, *bh = fp + 4 * kH, *wv = fp + 4 * kH + G.N3;
  const float bv = fpack[5 * kH + G.N3];
  float* vpart = reinterpret_cast<float*>(sm + G.off_part);  // [32][8]
  float* lpart = vpart + kRows * 8;                           // [32][S]
  uint8_t* a_smem = sm + G.off_a;
  const float* stage = reinterpret_cast<const float*>(sm + G.off_obs);
  const int64_t ntiles = (N + kRows - 1) / kRows;
  const bool elect = tid == 0;

  // the sub-tile's obs rows: one bulk copy when 16-byte sized and aligned, else plain loads
  auto issue_obs = [&](int64_t tile) {
    const int64_t r0 = tile * kRows;
    const int rows = (int)((N - r0) < kRows ? (N - r0) : kRows);
    const uint32_t bytes = (uint32_t)rows * G.obs_ld * 4;
    if ((bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(obs + r0 * G.obs_ld) & 15u) == 0) {
      if (elect) {
        mbar_expect_tx(bar_obs, bytes);
        bulk_g2s(s_base + G.off_obs, obs + r0 * G.obs_ld, bytes, bar_obs);
      }
      return true;
    }
    return false;
  };

  if (elect) {
    mbar_init(bar_w, 1);
    mbar_init(bar_obs, 1);
    mbar_init(bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: 512 columns (layer 1/2 at 0..255, the head at 0..N3-1 once they are consumed)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int64_t tile = blockIdx.x;
  bool bulk = tile < ntiles ? issue_obs(tile) : false;
  if (elect) {  // weights and float parameters: two bulk copies completing on one barrier
    mbar_expect_tx(bar_w, G.w_bytes + G.f_floats * 4);
    bulk_g2s(s_base, wpack, G.w_bytes, bar_w);
    bulk_g2s(s_base + G.off_f, fpack, G.f_floats * 4, bar_w);
  }
  const uint64_t key = mix64(seed ^ mix64(counter[0] + 0x9E3779B97F4A7C15ULL));
  uint32_t ph_obs = 0, ph_mma = 0;
  bool weights = false;

  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kRows;
    const int rows = (int)((N - r0) < kRows ? (N - r0) : kRows);
    if (bulk) {
      mbar_wait(bar_obs, ph_obs);
      ph_obs ^= 1;
    } else {
      float* st = reinterpret_cast<float*>(sm + G.off_obs);
      for (int i = tid; i < rows * G.obs_ld; i += kThreads) st[i] = obs[r0 * G.obs_ld + i];
      __syncthreads();
    }
    // obs (float32, row stride obs_ld) -> bf16 A operand [k/8][row][8], zero
    // past obs_dim and past the last row, written into all four replicas
    for (int it = tid; it < kRows * G.C1; it += kThreads) {
      const int c = it / kRows, r = it - c * kRows;
      const float* src = stage + r * G.obs_ld + 8 * c;
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (8 * c + j < G.obs_dim && r < rows) ? src[j] : 0.f;
      const uint4 val =
          make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
#pragma unroll
      for (int rep = 0; rep < 4; ++rep)
        *reinterpret_cast<uint4*>(a_smem + (size_t)c * (kM * 16) + (r + kRows * rep) * 16) = val;
    }
    fence_proxy_async();
    __syncthreads();
    // the staging area is free: the next sub-tile's obs copy overlaps this one's layers
    const int64_t nxt = tile + gridDim.x;
    if (nxt < ntiles) bulk = issue_obs(nxt);
    if (!weights) {
      mbar_wait(bar_w, 0);
      weights = true;
    }

    // layer 1: D[0:128) = A[128 x K1] W1^T
    if (elect) {
      tc_fence_after();
      mma_chain(tmem, s_base + G.off_a, kM * 16, s_base + G.off_w1, 2 * kH * 16, G.K1 / 16, idesc_bf16(kM, 2 * kH));
      mma_commit(bar_mma);
    }
    mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
    if (warp < 16) {  // h1 chunk `warp` (columns 8w..8w+7) of row `lane`
      uint32_t v[8];
      VYP_LD8(tmem + tq + 8 * warp, v, 0);
      tmem_wait_ld();
      act_to_a(v, b1 + 8 * warp, a_smem, warp, lane);
    }
    tc_fence_before();
    fence_proxy_async();
    __syncthreads();

    // layer 2: actor D[128:192) = h1a Wa2^T, critic D[192:256) = h1c Wc2^T
    if (elect) {
      tc_fence_after();
      mma_chain(tmem + 128, s_base + G.off_a, kM * 16, s_base + G.off_wa2, kH * 16, kH / 16, idesc_bf16(kM, kH));
      mma_chain(tmem + 192, s_base + G.off_a + 8 * kM * 16, kM * 16, s_base + G.off_wc2, kH * 16, kH / 16,
                idesc_bf16(kM, kH));
      mma_commit(bar_mma);
    }
    mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
    if (warp < 16) {
      uint32_t v[8];
      VYP_LD8(tmem + tq + 128 + 8 * warp, v, 0);
      tmem_wait_ld();
      if (warp < 8) {
        act_to_a(v, b2a + 8 * warp, a_smem, warp, lane);  // h2a -> A chunks 0..7
      } else {
        // value head: bf16 h2c times the bf16 value weights, fp32 partial sums
        const float* b = b2c + 8 * (warp - 8);
        const float* w = wv + 8 * (warp - 8);
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += bf16r(tanh_sfu(bf16r(__uint_as_float(v[j]) + b[j]))) * w[j];
        vpart[lane * 8 + (warp - 8)] = acc;
      }
    }
    tc_fence_before();
    fence_proxy_async();
    __syncthreads();

    // layer 3: head D[0:N3) = h2a Wh^T (two chains: N = n3a, n3b)
    if (elect) {
      tc_fence_after();
      mma_chain(tmem, s_base + G.off_a, kM * 16, s_base + G.off_wh, G.N3 * 16, kH / 16, idesc_bf16(kM, G.n3a));
      if (G.n3b > 0)
        mma_chain(tmem + G.n3a, s_base + G.off_a, kM * 16, s_base + G.off_wh + G.n3a * 16, G.N3 * 16, kH / 16,
                  idesc_bf16(kM, G.n3b));
      mma_commit(bar_mma);
    }
    const int64_t grow = r0 + lane;
    const bool live = lane < rows;
    if (warp == 16 && live) {  // idle during the head otherwise
      const float* vp = vpart + lane * 8;
      value[grow] = bf16r((((vp[0] + vp[1]) + (vp[2] + vp[3])) + ((vp[4] + vp[5]) + (vp[6] + vp[7]))) + bv);
    }
    mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
    for (int s = warp; s < G.S; s += kWarps) {
      uint32_t v[24];
      const uint32_t ta = tmem + tq + kSlotCols * s;
      VYP_LD16(ta, v);
      VYP_LD8(ta + 16, v, 16);
      tmem_wait_ld();
      // one uniform per (row, slot): element (row * S + s) of this call's stream
      const uint64_t x = mix64(key + (uint64_t)(grow * G.S + s) * 0x9E3779B97F4A7C15ULL);
      int a;
      float lp;
      if (G.A == kMaxA)
        sample_slot<kMaxA>(v, bh + kSlotCols * s, G.A, x, a, lp);
      else
        sample_slot<0>(v, bh + kSlotCols * s, G.A, x, a, lp);
      lpart[lane * G.S + s] = lp;
      if (live) {
        actions[grow * G.S + s] = (uint8_t)a;
        if (logits_out)
#pragma unroll
          for (int k = 0; k < kMaxA; ++k)
            if (k < G.A) logits_out[grow * (G.S * G.A) + s * G.A + k] = bf16r(__uint_as_float(v[k]) + bh[kSlotCols * s + k]);
      }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0 && live) {  // log-probability: slot terms summed in slot order
      float acc = 0.f;
      for (int s = 0; s < G.S; ++s) acc += lpart[lane * G.S + s];
      logp[grow] = acc;
    }
  }

  // teardown: release TMEM; the last CTA out advances the call counter
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (elect) {
    __threadfence();
    if (atomicAdd(counter + 1, 1ull) == gridDim.x - 1) {
      counter[1] = 0;
      counter[0] += 1;
      __threadfence();
    }
  }
}

thread_local std::string g_err;

}  // namespace vyp

extern "C" {

int vy_policy_geometry(int32_t obs_dim, int32_t obs_ld, int32_t S, int32_t A, int32_t out[4]) {
  if (obs_dim < 1 || obs_ld < obs_dim || vyp::ceil16(obs_dim) > vyp::kMaxK1 || obs_ld > vyp::kMaxK1 || S < 1 ||
      A < 2 || A > vyp::kMaxA || vyp::ceil16(S * vyp::kSlotCols) > 512 || S > 64)
    return VY_ERR_UNSUPPORTED;
  const vyp::Geo g = vyp::make_geo(obs_dim, obs_ld, S, A);
  out[0] = (int32_t)g.w_bytes;   // bf16 weight blob bytes
  out[1] = (int32_t)g.f_floats;  // float parameter count
  out[2] = g.N3;                 // head rows (slot s at rows 24s..24s+A-1)
  out[3] = (int32_t)g.smem;      // dynamic shared memory per CTA
  return VY_OK;
}

int vy_policy_step(const float* obs, int64_t obs_ld, int64_t N, int32_t obs_dim, int32_t S, int32_t A,
                   const void* wpack, const float* fpack, uint64_t seed, int64_t* counter, uint8_t* actions,
                   float* logp, float* value, float* logits_out, void* stream) {
  if (!obs || !wpack || !fpack || !counter || !actions || !logp || !value || N < 1) return VY_ERR_ARG;
  int32_t geo[4];
  if (vy_policy_geometry(obs_dim, (int32_t)obs_ld, S, A, geo) != VY_OK) return VY_ERR_UNSUPPORTED;
  if (((reinterpret_cast<uintptr_t>(wpack) | reinterpret_cast<uintptr_t>(fpack)) & 15u) != 0) return VY_ERR_ARG;
  const vyp::Geo g = vyp::make_geo(obs_dim, (int)obs_ld, S, A);
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(vyp::k_policy_step, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  const int64_t tiles = (N + vyp::kRows - 1) / vyp::kRows;
  const unsigned grid = (unsigned)(tiles < num_sms ? tiles : num_sms);
  vyp::k_policy_step<<<grid, vyp::kThreads, g.smem, (cudaStream_t)stream>>>(
      obs, N, g, static_cast<const uint8_t*>(wpack), fpack, seed, reinterpret_cast<unsigned long long*>(counter),
      actions, logp, value, logits_out);
  return cudaGetLastError() == cudaSuccess ? VY_OK : VY_ERR_CUDA;
}

}  // extern "C"
