// vy_kernels.cuh — sm_100a kernels: fused step, reset, fused T-step rollout,
// random actions, env seeding.
//
// One thread per env; 128-thread CTAs; grid = ceil(B / 128).  Per-CTA shared
// memory holds the car-profile table, the action->delta table and, for
// float32 observations, a per-warp staging tile: each thread writes its obs
// row into the tile (row stride obs_len is odd for the shipped layouts, so
// the 32 rows hit 32 distinct banks), then one lane streams the warp's
// 32 x obs_len block — contiguous in global memory — with a single bulk async
// copy (cp.async.bulk, the TMA bulk path) instead of 32 x obs_len strided
// scalar stores.
#pragma once

#include <climits>

#include "vy_step.cuh"

namespace vy {

constexpr int kBlock = 128;
constexpr int kWarps = kBlock / 32;

struct SmemLayout {
  int prof_off, dtab_off, obs_off, bytes, obs_tile;  // obs_tile: floats per warp (0 = no staging)
};

__host__ __device__ inline SmemLayout smem_layout(int k, int obs_len, bool stage) {
  SmemLayout L;
  L.prof_off = 0;
  L.dtab_off = kMaxProfiles * (int)sizeof(Profile);
  const int nd = (2 * k + 1) <= 255 ? (2 * k + 1) : 0;
  int off = L.dtab_off + nd * 8;
  off = (off + 127) & ~127;
  L.obs_off = off;
  L.obs_tile = stage ? 32 * obs_len : 0;
  L.bytes = off + kWarps * L.obs_tile * 4;
  return L;
}

template <int NP>
__device__ __forceinline__ void stage_tables(const Params<NP>& P, unsigned char* smem, const SmemLayout& L,
                                             const Profile*& prof, const double*& dtab) {
  Profile* sp = reinterpret_cast<Profile*>(smem + L.prof_off);
  double* sd = reinterpret_cast<double*>(smem + L.dtab_off);
  const double* gp = reinterpret_cast<const double*>(P.profiles);
  double* spd = reinterpret_cast<double*>(sp);
  for (int i = threadIdx.x; i < kMaxProfiles * 5; i += blockDim.x) spd[i] = __ldg(gp + i);
  const int nd = 2 * P.k + 1;
  if (nd <= 255)
    for (int i = threadIdx.x; i < nd; i += blockDim.x) sd[i] = __ldg(P.delta_tab + i);
  __syncthreads();
  prof = sp;
  dtab = nd <= 255 ? sd : nullptr;
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Emit one obs row per active thread.  Staged (float32): rows go to the warp's
// smem tile and a full warp issues one bulk copy; partial warps copy lane-wise.
template <int NP>
__device__ __forceinline__ void emit_obs(const Params<NP>& P, const Profile* prof, const Env<NP>& E, int64_t b,
                                         bool active, void* obs_base, float* tile, bool f64) {
  const int L = P.obs_len;
  if (f64) {
    if (active) write_obs(P, prof, E, reinterpret_cast<double*>(obs_base) + b * L);
    return;
  }
  float* gobs = reinterpret_cast<float*>(obs_base);
  if (!tile) {
    if (active) write_obs(P, prof, E, gobs + b * L);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t b0 = b - lane;
  const int64_t left = P.B - b0;
  const int rows = left >= 32 ? 32 : (int)left;
  if (lane == 0) bulk_wait_read();  // previous bulk copy out of this tile (rollout) has read it
  __syncwarp();
  if (active) write_obs(P, prof, E, tile + lane * L);
  fence_async_smem();
  __syncwarp();
  if (rows == 32) {
    if (lane == 0) bulk_store(gobs + b0 * L, tile, (uint32_t)(32 * L * 4));
  } else {
    for (int e = lane; e < rows * L; e += 32) gobs[b0 * L + e] = tile[e];
  }
}

template <int NP>
__global__ void __launch_bounds__(kBlock) k_step(const __grid_constant__ Params<NP> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemLayout Ls = smem_layout(P.k, P.obs_len, P.flags & 0x100u);
  const Profile* prof;
  const double* dtab;
  stage_tables(P, smem, Ls, prof, dtab);
  const int64_t b = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool active = b < P.B;
  const bool f64 = P.flags & VY_F_OUT_F64;
  float* tile = Ls.obs_tile ? reinterpret_cast<float*>(smem + Ls.obs_off) + (threadIdx.x >> 5) * Ls.obs_tile : nullptr;
  Env<NP> E;
  if (active) {
    load_env(P, b, E);
    const int dt = P.act_dtype;
    const int64_t rs = P.act_row, cs = P.act_col;
    auto act = [&](int slot) -> int {
      const int64_t at = b * rs + slot * cs;
      if (dt == VY_ACT_U8) return __ldg(reinterpret_cast<const uint8_t*>(P.actions) + at);
      if (dt == VY_ACT_I32) return __ldg(reinterpret_cast<const int32_t*>(P.actions) + at);
      const long long v = __ldg(reinterpret_cast<const long long*>(P.actions) + at);
      return v < INT_MIN ? INT_MIN : (v > INT_MAX ? INT_MAX : (int)v);
    };
    const StepResult r = step_env(P, prof, dtab, E, b, act);
    bool reset = false;
    if (r.done && (P.flags & VY_F_AUTO_RESET)) {
      const int ep = P.st.episode[b] + 1;
      reset_regs(P, E, P.st.env_seed[b], ep, nullptr, b);
      P.st.episode[b] = ep;
      reset = true;
    }
    store_env(P, b, E, reset);
    if (f64)
      reinterpret_cast<double*>(P.out.reward)[b] = r.reward;
    else
      reinterpret_cast<float*>(P.out.reward)[b] = (float)r.reward;
    P.out.done[b] = r.done;
  }
  emit_obs(P, prof, E, b, active, P.out.obs, tile, f64);
  if (tile && (threadIdx.x & 31) == 0) bulk_wait_read();
}

template <int NP>
__global__ void __launch_bounds__(kBlock) k_reset(const __grid_constant__ Params<NP> P, const uint8_t* mask,
                                                  int episode_mode, const int32_t* inj_day) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemLayout Ls = smem_layout(P.k, P.obs_len, false);
  const Profile* prof;
  const double* dtab;
  stage_tables(P, smem, Ls, prof, dtab);
  const int64_t b = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  if (b >= P.B || (mask && !mask[b])) return;
  Env<NP> E;
  const int ep = episode_mode ? P.st.episode[b] + 1 : 0;
  reset_regs(P, E, P.st.env_seed[b], ep, inj_day, b);
  P.st.episode[b] = ep;
  store_env(P, b, E, true);
  if (P.flags & VY_F_OUT_F64)
    write_obs(P, prof, E, reinterpret_cast<double*>(P.out.obs) + b * P.obs_len);
  else
    write_obs(P, prof, E, reinterpret_cast<float*>(P.out.obs) + b * P.obs_len);
}

// RandomPolicy stream draw: row key k, overall draw number j (1-based)
__device__ __forceinline__ int policy_action(uint64_t key, uint64_t j, int hi) {
  const double u = __dmul_rn((double)(mix64(key + j * kGolden) >> 11), 1.0 / 9007199254740992.0);
  const int a = (int)__double2ll_rz(__dmul_rn(u, (double)hi));
  return a >= hi ? hi - 1 : a;
}

// Fused T-step rollout: state stays in registers across steps, actions come
// from the in-kernel RandomPolicy stream, obs/reward/done are emitted every
// step, done envs auto-reset in place.
template <int NP>
__global__ void __launch_bounds__(kBlock) k_rollout(const __grid_constant__ Params<NP> P, int T,
                                                    uint64_t policy_seed, int64_t index0, int64_t call0,
                                                    int64_t obs_stride, int64_t rew_stride) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemLayout Ls = smem_layout(P.k, P.obs_len, P.flags & 0x100u);
  const Profile* prof;
  const double* dtab;
  stage_tables(P, smem, Ls, prof, dtab);
  const int64_t b = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool active = b < P.B;
  const bool f64 = P.flags & VY_F_OUT_F64;
  float* tile = Ls.obs_tile ? reinterpret_cast<float*>(smem + Ls.obs_off) + (threadIdx.x >> 5) * Ls.obs_tile : nullptr;
  Env<NP> E;
  uint64_t pkey = 0;
  int episode = 0;
  if (active) {
    load_env(P, b, E);
    pkey = fold(fold(fold(kKey0, policy_seed), (uint64_t)(index0 + b)), 2);
    episode = P.st.episode[b];
  }
  const int ns = P.n_ports + 1, hi = 2 * P.k + 1;
  for (int t = 0; t < T; ++t) {
    double rew = 0.0;
    bool done = false;
    if (active) {
      const uint64_t j0 = (uint64_t)(call0 + t) * (uint64_t)ns;
      auto act = [&](int slot) -> int { return policy_action(pkey, j0 + slot + 1, hi); };
      const StepResult r = step_env(P, prof, dtab, E, b, act);
      rew = r.reward;
      done = r.done;
      if (done) {
        ++episode;
        reset_regs(P, E, P.st.env_seed[b], episode, nullptr, b);
      }
      if (f64)
        reinterpret_cast<double*>(P.out.reward)[t * rew_stride + b] = rew;
      else
        reinterpret_cast<float*>(P.out.reward)[t * rew_stride + b] = (float)rew;
      P.out.done[t * rew_stride + b] = done;
    }
    void* obs_t = f64 ? (void*)(reinterpret_cast<double*>(P.out.obs) + t * obs_stride)
                      : (void*)(reinterpret_cast<float*>(P.out.obs) + t * obs_stride);
    emit_obs(P, prof, E, b, active, obs_t, tile, f64);
  }
  if (tile && (threadIdx.x & 31) == 0) bulk_wait_read();
  if (active) {
    store_env(P, b, E, true);
    P.st.episode[b] = episode;
  }
}

}  // namespace vy
