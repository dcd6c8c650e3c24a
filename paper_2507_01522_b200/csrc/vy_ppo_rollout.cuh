// vy_ppo_rollout.cuh — the whole PPO rollout (T policy passes, T env steps and
// the bootstrap value) as ONE persistent kernel, for the small batches the
// paper trains on (16 envs).
//
// The per-step path is a CUDA graph of 2T+1 launches: vy_policy_step (tcgen05
// MLP, one CTA per 32 rows) then the one-warp-per-env step (k_rollout_wide
// with T = 1).  At 16 envs each launch is a few microseconds of dependent
// latency on one or two SMs and the policy kernel re-stages ~100 KB of weights
// and re-allocates TMEM every step; the measured step is ~24 us.  Here each CTA
// owns epc envs (2..16, one env warp each) for all T steps:
//   setup: TMEM allocated once, the bf16 weights bulk-copied into shared
//     memory once, the station tables staged once, env warp w loads env
//     b0 + w into registers (WideEnv: lane = port);
//   per step t: obs rows (shared, float32) -> bf16 A operand -> the policy's
//     three tcgen05 layers and epilogues (the SAME instructions, operand
//     layouts, epilogue arithmetic and sampling stream as k_policy_step, so
//     actions / log-probabilities / values are bit-identical to the per-step
//     path) -> actions into shared memory and the rollout buffer -> env warp
//     w steps env b0 + w with them (WideEnv::step, bit-identical to
//     k_rollout_wide) and writes the next obs row to the rollout buffer and
//     to the shared staging rows the next policy pass reads;
//   after step T-1: one more policy pass = the bootstrap value of obs[T];
//   teardown: env state back to HBM, TMEM released, the last CTA out
//     advances the sampler's call counter by T + 1 (one per policy pass, as
//     T + 1 vy_policy_step calls would).
// Envs are independent, so CTAs never synchronise with each other; a batch
// of B envs is ceil(B / epc) CTAs (one per SM: ~175 KB of shared memory),
// epc = clamp(ceil(B / #SMs), 2, 16) chosen by vy_ppo_rollout: the policy
// pass costs the same for 1 or 16 rows, fewer env warps per SM step faster.
// 16 envs: 6.9 us per step (policy pass ~8k cycles, env step ~5.4k).
#pragma once

#include "vy_umma.cuh"
#include "vy_wide.cuh"

namespace vy {

constexpr int kPpoEnvs = 16;   // max envs (= env warps) per CTA
constexpr int kPpoWarps = 16;  // warp w: h1 chunk w, actor/critic chunk w, head slots w, w + 16, ...
constexpr int kPpoThreads = 32 * kPpoWarps;
constexpr int kPpoActRow = 64;  // bytes per env of the shared action rows

struct PpoBufs {
  const uint8_t* wpack;  // bf16 weights, UMMA layout (pack_policy)
  const float* fpack;    // biases, value weights (pack_policy)
  uint64_t seed;
  unsigned long long* counter;  // {call, CTAs done}
  float* obs;                   // [T+1][B][obs_len]: row 0 read, rows 1..T written
  uint8_t* actions;             // [T][B][S]
  float* logp;                  // [T][B]
  float* value;                 // [T+1][B]
};

// shared memory: station tables | env scratch | action rows | (1 KB aligned) policy area (vyp::Geo)
__host__ __device__ inline uint32_t ppo_scratch_off(int n_profiles, int k, int n_ports, int n_nodes) {
  return (uint32_t)tables_bytes(n_profiles, k, n_ports, n_nodes);
}
__host__ __device__ inline uint32_t ppo_acts_off(uint32_t scratch) {
  return scratch + kPpoEnvs * kWideScratch * 8;
}
__host__ __device__ inline uint32_t ppo_policy_off(uint32_t scratch) {
  return (ppo_acts_off(scratch) + kPpoEnvs * kPpoActRow + 1023) & ~1023u;
}

#ifdef VY_PPO_PROF  // phase timing build (scripts/probe_ppo_phases.py): clock64 deltas of CTA 0 thread 0
__device__ unsigned long long g_ppo_prof[16];
#define PPO_MARK(i)                                   \
  if (blockIdx.x == 0 && threadIdx.x == 0) {          \
    const unsigned long long now_ = clock64();        \
    g_ppo_prof[i] += now_ - prof_last;                \
    prof_last = now_;                                 \
  }
#else
#define PPO_MARK(i)
#endif

template <int M>
__global__ void __launch_bounds__(kPpoThreads, 1)
    k_ppo_rollout(const __grid_constant__ Params P, int T, int epc, const vyp::Geo G, const PpoBufs R) {
  using vyp::kH;
  using vyp::kM;
  using vyp::kRows;
  using vyp::kSlotCols;
  using vyp::kMaxA;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t scr = ppo_scratch_off(P.n_profiles, P.k, P.n_ports, P.n_nodes);
  double* scratch = reinterpret_cast<double*>(vy_smem + scr) + warp * kWideScratch;
  uint8_t* act_s = vy_smem + ppo_acts_off(scr);
  uint8_t* sm = vy_smem + ppo_policy_off(scr);
  const uint32_t tq = (uint32_t)(32 * (warp & 3)) << 16;  // this warp's TMEM lane quadrant
  const uint32_t s_base = vyp::smem_u32(sm);
  const uint32_t bar_w = s_base + G.off_bar, bar_mma = bar_w + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + G.off_bar + 24);
  float* fp = reinterpret_cast<float*>(sm + G.off_f);
  const float *b1 = fp, *b2a = fp + 2 * kH, *b2c = fp + 3 * kH, *bh = fp + 4 * kH, *wv = fp + 4 * kH + G.N3;
  const float bv = R.fpack[5 * kH + G.N3];
  float* vpart = reinterpret_cast<float*>(sm + G.off_part);  // [32][8]
  float* lpart = vpart + kRows * 8;                           // [32][S]
  uint8_t* a_smem = sm + G.off_a;
  float* stage = reinterpret_cast<float*>(sm + G.off_obs);  // obs rows, float32, stride obs_ld
  const bool elect = tid == 0;
  const int64_t B = P.B, b0 = (int64_t)blockIdx.x * epc;
  const int rows = (int)((B - b0) < epc ? (B - b0) : epc);  // this CTA's envs (epc <= 16)
  const int n = P.n_ports, OL = P.obs_len;

  if (elect) {
    vyp::mbar_init(bar_w, 1);
    vyp::mbar_init(bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: 512 columns for the whole rollout (layers 1/2 at 0..255, the head at 0..N3-1)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(vyp::smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // obs[0] rows of this CTA's envs -> staging rows
  for (int i = tid; i < rows * OL; i += kPpoThreads) {
    const int r = i / OL, c = i - r * OL;
    stage[r * G.obs_ld + c] = R.obs[(b0 + r) * OL + c];
  }
  Prof prof;
  PortC pc;
  TreeC tc;
  const double* dtab;
  vyp::tc_fence_before();
  stage_tables(P, prof, dtab, pc, tc);  // ends in __syncthreads: barriers, TMEM address and obs rows visible
  vyp::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (elect) {  // weights and float parameters: two bulk copies completing on one barrier, once per rollout
    vyp::mbar_expect_tx(bar_w, G.w_bytes + G.f_floats * 4);
    vyp::bulk_g2s(s_base, R.wpack, G.w_bytes, bar_w);
    vyp::bulk_g2s(s_base + G.off_f, R.fpack, G.f_floats * 4, bar_w);
  }
  const bool env_warp = warp < rows;
  WideEnv<M> env;
  if (env_warp) env.load(P, pc, dtab, b0 + warp, lane);
  const unsigned long long call0 = R.counter[0];
  uint32_t ph_mma = 0;

#ifdef VY_PPO_PROF
  unsigned long long prof_last = clock64();
#endif
  for (int t = 0;; ++t) {
    PPO_MARK(0);
    // the sampler key of policy pass t (k_policy_step's key of call call0 + t)
    const uint64_t key = vyp::mix64(R.seed ^ vyp::mix64(call0 + (unsigned long long)t + 0x9E3779B97F4A7C15ULL));
    // obs rows -> bf16 A operand [k/8][row][8], zero past obs_dim and past the last row, 4 replicas
    for (int it = tid; it < kRows * G.C1; it += kPpoThreads) {
      const int c = it / kRows, r = it - c * kRows;
      const float* src = stage + r * G.obs_ld + 8 * c;
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (8 * c + j < G.obs_dim && r < rows) ? src[j] : 0.f;
      const uint4 val =
          make_uint4(vyp::pack_bf16(x[0], x[1]), vyp::pack_bf16(x[2], x[3]), vyp::pack_bf16(x[4], x[5]), vyp::pack_bf16(x[6], x[7]));
#pragma unroll
      for (int rep = 0; rep < 4; ++rep)
        *reinterpret_cast<uint4*>(a_smem + (size_t)c * (kM * 16) + (r + kRows * rep) * 16) = val;
    }
    vyp::fence_proxy_async();
    __syncthreads();
    if (t == 0) vyp::mbar_wait(bar_w, 0);
    PPO_MARK(1);

    // layer 1: D[0:128) = A[128 x K1] W1^T
    if (elect) {
      vyp::tc_fence_after();
      vyp::mma_chain(tmem, s_base + G.off_a, kM * 16, s_base + G.off_w1, 2 * kH * 16, G.K1 / 16, vyp::idesc_bf16(kM, 2 * kH));
      vyp::mma_commit(bar_mma);
    }
    vyp::mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    PPO_MARK(2);
    vyp::tc_fence_after();
    {  // h1 chunk `warp` (columns 8w..8w+7) of row `lane`
      uint32_t v[8];
      VYP_LD8(tmem + tq + 8 * warp, v, 0);
      vyp::tmem_wait_ld();
      vyp::act_to_a(v, b1 + 8 * warp, a_smem, warp, lane);
    }
    vyp::tc_fence_before();
    vyp::fence_proxy_async();
    __syncthreads();
    PPO_MARK(3);

    // layer 2: actor D[128:192) = h1a Wa2^T, critic D[192:256) = h1c Wc2^T
    if (elect) {
      vyp::tc_fence_after();
      vyp::mma_chain(tmem + 128, s_base + G.off_a, kM * 16, s_base + G.off_wa2, kH * 16, kH / 16, vyp::idesc_bf16(kM, kH));
      vyp::mma_chain(tmem + 192, s_base + G.off_a + 8 * kM * 16, kM * 16, s_base + G.off_wc2, kH * 16, kH / 16,
                vyp::idesc_bf16(kM, kH));
      vyp::mma_commit(bar_mma);
    }
    vyp::mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    PPO_MARK(4);
    vyp::tc_fence_after();
    {
      uint32_t v[8];
      VYP_LD8(tmem + tq + 128 + 8 * warp, v, 0);
      vyp::tmem_wait_ld();
      if (warp < 8) {
        vyp::act_to_a(v, b2a + 8 * warp, a_smem, warp, lane);  // h2a -> A chunks 0..7
      } else {
        // value head: bf16 h2c times the bf16 value weights, fp32 partial sums
        const float* b = b2c + 8 * (warp - 8);
        const float* w = wv + 8 * (warp - 8);
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += vyp::bf16r(vyp::tanh_sfu(vyp::bf16r(__uint_as_float(v[j]) + b[j]))) * w[j];
        vpart[lane * 8 + (warp - 8)] = acc;
      }
    }
    vyp::tc_fence_before();
    vyp::fence_proxy_async();
    __syncthreads();
    PPO_MARK(5);

    // layer 3: head D[0:N3) = h2a Wh^T (two chains: N = n3a, n3b)
    if (elect) {
      vyp::tc_fence_after();
      vyp::mma_chain(tmem, s_base + G.off_a, kM * 16, s_base + G.off_wh, G.N3 * 16, kH / 16, vyp::idesc_bf16(kM, G.n3a));
      if (G.n3b > 0)
        vyp::mma_chain(tmem + G.n3a, s_base + G.off_a, kM * 16, s_base + G.off_wh + G.n3a * 16, G.N3 * 16, kH / 16,
                  vyp::idesc_bf16(kM, G.n3b));
      vyp::mma_commit(bar_mma);
    }
    const int64_t grow = b0 + lane;
    const bool live = lane < rows;
    if (warp == kPpoWarps - 1 && live) {  // the value, while the head MMAs run
      const float* vp = vpart + lane * 8;
      R.value[t * B + grow] = vyp::bf16r((((vp[0] + vp[1]) + (vp[2] + vp[3])) + ((vp[4] + vp[5]) + (vp[6] + vp[7]))) + bv);
    }
    vyp::mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1;
    PPO_MARK(6);
    vyp::tc_fence_after();
    const bool sample = t < T;  // pass T is the bootstrap value only
    // the head: rows 0..15 are this CTA's envs (TMEM lanes 0..15 of every
    // quadrant), so a warp takes two slots at once — lanes 0..15 slot s0,
    // lanes 16..31 slot s0 + 8 through the .16x32bx2 load — and 17 slots
    // occupy 9 warps for one round (warp w < 8: slots w, w + 8; warp w >= 8:
    // slot w + 8 and, for S > 24, w + 16)
    const int hrow = lane & 15;
    const int64_t hgrow = b0 + hrow;
    for (int s0 = warp < 8 ? warp : warp + 8; sample && s0 < G.S; s0 += 32) {
      const bool pair = s0 + 8 < G.S;  // warp-uniform
      uint32_t v[24];
      const uint32_t ta = tmem + tq + kSlotCols * s0;
      if (pair) {
        VYP_LD16X2(ta, v, 192);  // 192 = 8 * kSlotCols columns: slot s0 + 8
        VYP_LD8X2(ta + 16, v, 16, 192);
      } else {
        VYP_LD16(ta, v);
        VYP_LD8(ta + 16, v, 16);
      }
      vyp::tmem_wait_ld();
      const int s = (pair && lane >= 16) ? s0 + 8 : s0;
      const bool mine = lane < 16 || pair;  // an unpaired warp's upper lanes hold unused rows
      // one uniform per (row, slot): element (row * S + s) of this pass's stream
      const uint64_t x = vyp::mix64(key + (uint64_t)(hgrow * G.S + s) * 0x9E3779B97F4A7C15ULL);
      int a;
      float lp;
      if (G.A == kMaxA)
        vyp::sample_slot<kMaxA>(v, bh + kSlotCols * s, G.A, x, a, lp);
      else
        vyp::sample_slot<0>(v, bh + kSlotCols * s, G.A, x, a, lp);
      if (mine) {
        lpart[hrow * G.S + s] = lp;
        if (hrow < rows) {
          R.actions[(t * B + hgrow) * G.S + s] = (uint8_t)a;
          act_s[hrow * kPpoActRow + s] = (uint8_t)a;
        }
      }
    }
    vyp::tc_fence_before();
    __syncthreads();
    PPO_MARK(7);
    if (!sample) break;
    if (warp == kPpoWarps - 1 && live) {  // log-probability: slot terms summed in slot order (off the env warps
      float acc = 0.f;                      // unless the CTA has 16 envs)
      for (int s = 0; s < G.S; ++s) acc += lpart[lane * G.S + s];
      R.logp[t * B + grow] = acc;
    }
    PPO_MARK(8);
    // env step t on the env warps: next obs -> rollout row t + 1 and the staging row
    if (env_warp) {
      const int a = lane < n ? act_s[warp * kPpoActRow + lane] : P.k;
      env.template step<true>(P, prof, tc, lane, a, R.obs + ((int64_t)(t + 1) * B + b0 + warp) * OL,
                              stage + warp * G.obs_ld, (int64_t)t * B + b0 + warp, scratch, scratch + 32);
    }
    PPO_MARK(9);
    __syncthreads();
  }
  if (env_warp) env.store(P, lane);

  // teardown: release TMEM; the last CTA out advances the call counter by the T + 1 passes
  if (warp == 0) {
    vyp::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (elect) {
    __threadfence();
    if (atomicAdd(R.counter + 1, 1ull) == gridDim.x - 1) {
      R.counter[1] = 0;
      R.counter[0] += (unsigned long long)T + 1;
      __threadfence();
    }
  }
}

}  // namespace vy
