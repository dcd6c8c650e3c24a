// vy_umma.cuh — the policy network's tensor-core building blocks (sm_100a):
// shared-memory geometry, mbarrier / bulk-copy / tcgen05 PTX wrappers, the
// UMMA descriptors and the bf16 epilogue helpers.  Used by the per-step
// policy kernel (vy_policy.cu) and the fused PPO rollout (vy_ppo_rollout.cuh),
// so both run the same instructions on the same operand layouts.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace vyp {

constexpr int kWarps = 17;     // warp w: A chunk w of epilogues 1/2 (w < 16), action slot w of the head
constexpr int kThreads = 32 * kWarps;
constexpr int kRows = 32;      // unique rows per MMA tile (replicated 4x into M = 128)
constexpr int kM = 128;        // rows per tile (UMMA M)
constexpr int kH = 64;         // hidden width per branch
constexpr int kSlotCols = 24;  // TMEM / head-row columns per action slot
constexpr int kMaxK1 = 128;    // padded observation width
constexpr int kMaxA = 21;      // actions per slot (2K+1 of the default K = 10)

__host__ __device__ constexpr int ceil16(int x) { return (x + 15) / 16 * 16; }

struct Geo {
  int K1, C1;        // padded obs width (multiple of 16), its 8-column chunks
  int N3, n3a, n3b;  // head width (S * kSlotCols padded to 16) and its two MMA widths
  int obs_ld, obs_dim, S, A;
  uint32_t off_w1, off_wa2, off_wc2, off_wh, w_bytes;  // weight blob (bf16, UMMA layout)
  uint32_t off_f;      // float params: b1[2H] b2a[H] b2c[H] bh[N3] wv[H] bv
  uint32_t f_floats;
  uint32_t off_a;      // A operand [16][128][8] bf16
  uint32_t off_obs;    // obs staging 128 x obs_ld float32
  uint32_t off_part;   // vpart[32][8], lpart[32][S] float32
  uint32_t off_bar;    // mbarriers: weights, obs, mma; TMEM base address
  uint32_t smem;
};

__host__ __device__ inline Geo make_geo(int obs_dim, int obs_ld, int S, int A) {
  Geo g{};
  g.obs_dim = obs_dim;
  g.obs_ld = obs_ld;
  g.S = S;
  g.A = A;
  g.K1 = ceil16(obs_dim);
  g.C1 = g.K1 / 8;
  g.N3 = ceil16(S * kSlotCols);
  g.n3a = g.N3 > 256 ? 256 : g.N3;
  g.n3b = g.N3 - g.n3a;
  g.off_w1 = 0;
  g.off_wa2 = g.off_w1 + g.C1 * 2 * kH * 16;
  g.off_wc2 = g.off_wa2 + 8 * kH * 16;
  g.off_wh = g.off_wc2 + 8 * kH * 16;
  g.w_bytes = g.off_wh + 8 * g.N3 * 16;
  g.off_f = g.w_bytes;
  g.f_floats = 2 * kH + kH + kH + g.N3 + kH + 4;  // a multiple of 4: one 16-byte-sized bulk copy
  g.off_a = (g.off_f + g.f_floats * 4 + 127) & ~127u;
  g.off_obs = g.off_a + 16 * kM * 16;
  g.off_part = (g.off_obs + kRows * obs_ld * 4 + 15) & ~15u;
  g.off_bar = (g.off_part + kRows * (8 + S) * 4 + 15) & ~15u;
  g.smem = g.off_bar + 64;
  return g;
}

// ---- PTX wrappers ----------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// bulk async copy global -> shared (TMA engine), completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle: 8-row x 16-byte core
// matrices; LBO = byte stride between the two 8-element K chunks of one MMA,
// SBO = byte stride between 8-row groups (here 128: rows are 16 bytes apart).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor kind::f16: bf16 A/B, f32 accumulate, K-major A and B
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D = sum over k-steps of A[:, 16k:16k+16] B[:, 16k:16k+16]^T
__device__ __forceinline__ void mma_chain(uint32_t d_tmem, uint32_t a, uint32_t a_lbo, uint32_t b, uint32_t b_lbo,
                                          int ksteps, uint32_t idesc) {
  for (int k = 0; k < ksteps; ++k)
    mma_bf16(d_tmem, sdesc(a + 2 * k * a_lbo, a_lbo, 128), sdesc(b + 2 * k * b_lbo, b_lbo, 128), idesc, k > 0);
}

#define VYP_LD32(taddr, v)                                                                                          \
  asm volatile(                                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),           \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),     \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),   \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])    \
      : "r"(taddr))
#define VYP_LD16(taddr, v)                                                                                   \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),          \
                 "=r"(v[15])                                                                                      \
               : "r"(taddr))
#define VYP_LD8(taddr, v, o)                                                                                 \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                     \
               : "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), \
                 "=r"(v[o + 6]), "=r"(v[o + 7])                                                              \
               : "r"(taddr))
// 16 TMEM lanes, two column ranges: threads 0..15 read lanes 0..15 of the
// warp's quadrant at columns [c, c+n), threads 16..31 the same lanes at
// [c + off, c + off + n) (the .16x32bx2 shape; `off` an immediate)
#define VYP_LD16X2(taddr, v, off)                                                                             \
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16], " #off ";"                                                                             \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),          \
                 "=r"(v[15])                                                                                      \
               : "r"(taddr))
#define VYP_LD8X2(taddr, v, o, off)                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], " #off ";"             \
               : "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), \
                 "=r"(v[o + 6]), "=r"(v[o + 7])                                                              \
               : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// float -> bf16 (round to nearest even) -> float on the integer pipe: the
// same value as __float2bfloat16_rn for every non-NaN input (overflow to
// infinity included); NaN passes through unchanged
__device__ __forceinline__ float bf16r(float x) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  return x != x ? x : __uint_as_float(r);
}
// hardware tanh (MUFU.TANH, rel. error ~2^-11): its result is rounded to bf16 next
__device__ __forceinline__ float tanh_sfu(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float exp2_sfu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// two values rounded to bf16 (RNE) and back to float with one packed
// conversion (cvt.rn.bf16x2.f32) and two unpacks
__device__ __forceinline__ void bf16r2(float a, float b, float& ra, float& rb) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  ra = __low2float(p);
  rb = __high2float(p);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&p);
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// 8 accumulator columns of this thread's row -> bf16(tanh(bf16(acc + bias)))
// (cuBLAS bf16 output, then the bf16 tanh) -> one 16-byte A-operand chunk,
// stored into all four row replicas
__device__ __forceinline__ void act_to_a(const uint32_t* v, const float* bias, uint8_t* a_base, int c, int r) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float y0, y1;
    bf16r2(__uint_as_float(v[2 * j]) + bias[2 * j], __uint_as_float(v[2 * j + 1]) + bias[2 * j + 1], y0, y1);
    w[j] = pack_bf16(tanh_sfu(y0), tanh_sfu(y1));
  }
  const uint4 val = make_uint4(w[0], w[1], w[2], w[3]);
#pragma unroll
  for (int rep = 0; rep < 4; ++rep)
    *reinterpret_cast<uint4*>(a_base + (size_t)c * (kM * 16) + (r + kRows * rep) * 16) = val;
}

// One (row, slot) of the multi-discrete head: bf16 logits z = bf16(acc +
// bias) for the slot's A actions, max, exp(z - m) summed in action order, the
// inverse-CDF sample of the uniform `x >> 41` (the first k whose running sum
// passes u * sum; the last action if rounding leaves the target at or above
// the total) and its log-probability (z_a - m) - log(sum).  v: the slot's 24
// accumulator columns; bias: its 24 head biases (16-byte aligned).  AC: the
// action count at compile time (0 = runtime A).  Shared by k_policy_step and
// k_ppo_rollout so both sample identically.
template <int AC>
__device__ __forceinline__ void sample_slot(const uint32_t* v, const float* bias, int A_rt, uint64_t x, int& act,
                                            float& lp) {
  constexpr float kLog2e = 1.4426950408889634f;
  const int A = AC ? AC : A_rt;
  float bq[kSlotCols];
#pragma unroll
  for (int q = 0; q < kSlotCols / 4; ++q) {  // six 16-byte loads, all issued before use
    const float4 f = reinterpret_cast<const float4*>(bias)[q];
    bq[4 * q] = f.x;
    bq[4 * q + 1] = f.y;
    bq[4 * q + 2] = f.z;
    bq[4 * q + 3] = f.w;
  }
  constexpr int KN = AC ? AC : kMaxA;
  float z[KN + 1], e[KN];
#pragma unroll
  for (int k = 0; k < KN; k += 2)  // bf16 logits, two per packed conversion (v / bq have 24 entries)
    bf16r2(__uint_as_float(v[k]) + bq[k], __uint_as_float(v[k + 1]) + bq[k + 1], z[k], z[k + 1]);
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < KN; ++k) {
    if (!(AC || k < A)) z[k] = -INFINITY;
    m = fmaxf(m, z[k]);
  }
  const float mb = m * kLog2e;
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < KN; ++k) {
    e[k] = exp2_sfu(fmaf(z[k], kLog2e, -mb));  // exp(z - m); 0 past A
    sum += e[k];
  }
  const float target = ((float)(x >> 41) + 0.5f) * (1.f / 8388608.f) * sum;
  float c = 0.f, za = z[0];
  int a = -1;
#pragma unroll
  for (int k = 0; k < KN; ++k) {
    c += e[k];
    const bool take = a < 0 && (AC || k < A) && (target < c || k == A - 1);
    a = take ? k : a;
    za = take ? z[k] : za;
  }
  act = a;
  lp = (za - m) - __logf(sum);
}

}  // namespace vyp
