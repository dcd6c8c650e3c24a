// vy_kernels.cuh — sm_100a kernels over warp tiles.
//
//   k_step     one transition of every env (+ in-kernel auto-reset)
//   k_rollout  T transitions with in-kernel RandomPolicy actions, the tile's
//              state resident in shared memory for all T steps
//   k_reset    (masked) reset_env of every env
//
// CTA = W warps (W chosen on the host to fill shared memory); warp w of CTA
// c owns tile c*W + w (32 consecutive envs).  Per-CTA shared memory: the car
// profile table and the action->delta table, then W warp tiles.
#pragma once

#include <climits>

#include "vy_tile.cuh"

namespace vy {

constexpr int kProfileWords = (int)(sizeof(Profile) / 8);
// per-CTA table area: live car profiles, the (a-k)/k action grid, the per-port constants
__host__ __device__ inline int grid_table_off(int n_profiles) { return n_profiles * (int)sizeof(Profile); }
__host__ __device__ inline int portc_off(int n_profiles, int k) {
  const int nd = (2 * k + 1) <= 256 ? (2 * k + 1) : 0;
  return (grid_table_off(n_profiles) + nd * 8 + 15) & ~15;
}
__host__ __device__ inline int treec_off(int n_profiles, int k, int n_ports) {
  return portc_off(n_profiles, k) + n_ports * 8 * kPortWords;
}
__host__ __device__ inline int tables_bytes(int n_profiles, int k, int n_ports, int n_nodes) {
  return (treec_off(n_profiles, k, n_ports) + n_nodes * 32 + 127) & ~127;
}

__device__ __forceinline__ void stage_tables(const Params& P, Prof& prof, const double*& dtab, PortC& pc,
                                             TreeC& tc) {
  unsigned char* smem = vy_smem;
  double* spd = reinterpret_cast<double*>(smem);
  const double* gp = reinterpret_cast<const double*>(P.profiles);
  for (int i = threadIdx.x; i < P.n_profiles * kProfileWords; i += blockDim.x) spd[i] = __ldg(gp + i);
  double* sd = reinterpret_cast<double*>(smem + grid_table_off(P.n_profiles));
  const int nd = 2 * P.k + 1;
  if (nd <= 256)
    for (int i = threadIdx.x; i < nd; i += blockDim.x) sd[i] = __ldg(P.delta_tab + i);
  const int po = portc_off(P.n_profiles, P.k);
  double* sp = reinterpret_cast<double*>(smem + po);
  for (int i = threadIdx.x; i < P.n_ports * kPortWords; i += blockDim.x) sp[i] = __ldg(P.portc + i);
  const int to = treec_off(P.n_profiles, P.k, P.n_ports);
  double* st = reinterpret_cast<double*>(smem + to);
  for (int i = threadIdx.x; i < P.n_nodes * 4; i += blockDim.x) st[i] = __ldg(P.treec + i);
  __syncthreads();
  prof = Prof{smem_base()};
  pc = PortC{smem_base() + (uint32_t)po};
  tc = TreeC{smem_base() + (uint32_t)to};
  dtab = nd <= 256 ? sd : nullptr;
}

// Fused RandomPolicy (policies.py:51-73, rng.py:154-170): this lane's n+1
// actions of call `call` into its staged action row, computed while the
// tile's state copies are in flight.  Row b draws from stream_key(seed,
// index0 + b, 2); draw j = call*(n+1) + s + 1 is mix64(key + j*GOLDEN).
// With P.pol_out the warp also writes its [32][n+1] block to global memory.
__device__ __forceinline__ void policy_row(const Params& P, uint32_t tile, int64_t b0, int lane, int64_t call) {
  const int ns = P.n_ports + 1, hi = 2 * P.k + 1;
  const int64_t b = b0 + lane;
  const uint64_t key = fold(fold(fold(kKey0, P.pol_seed), (uint64_t)(P.pol_index0 + b)), 2);
  uint64_t kj = key + ((uint64_t)call * (uint64_t)ns + 1) * kGolden;
  const uint32_t row = smem_base() + tile + P.L.acts + lane * ns;
  for (int s = 0; s < ns; ++s, kj += kGolden) sts_u8(row + s, (uint32_t)policy_action(kj, 0, hi));
  if (P.pol_out) {
    __syncwarp();
    const int64_t left = P.B - b0;
    const int bytes = (left >= 32 ? 32 : (int)left) * ns;
    const unsigned char* src = vy_smem + tile + P.L.acts;
    uint8_t* g = P.pol_out + b0 * ns;
    if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
      for (int o = lane * 16; o < bytes; o += 512)
        *reinterpret_cast<uint4*>(g + o) = *reinterpret_cast<const uint4*>(src + o);
    } else {
      for (int o = lane; o < bytes; o += 32) g[o] = src[o];
    }
  }
}

// One step of the 32 envs of the tile starting at env b0.  Every lane runs
// the transition (padding lanes on their harmless padding columns, side
// effects masked) because the fused port loop synchronises the warp.
template <int M>
__device__ __forceinline__ void step_tile(const Params& P, Prof prof, const double* dtab, PortC pc, TreeC tc,
                                          uint32_t tile, int64_t b0, int lane, WarpBar& wb,
                                          unsigned long long* claim = nullptr, int64_t pol_call = 0,
                                          unsigned long long* claim_ctr = nullptr) {
  using C = Spec<M>;
  const Lane T = make_lane(P, tile, lane);
  const int64_t b = b0 + lane;
  const bool active = b < P.B;
  EnvRegs E{};  // zero for padding lanes so table lookups stay in bounds
  if (active) load_env<M>(P, b, E);
  // Two-stage tile load (tile_issue_meta / tile_issue_ports): the meta bytes
  // and action rows first, then the slots of the ports some env of the tile
  // occupies.  At night most ports are empty in every lane and are neither
  // read nor written (-12% step time); at the afternoon peak every port is
  // occupied somewhere and the extra round trip costs ~3% (day average -1.5%).
  tile_issue_meta(P, tile, b0, lane, C::staged(P) && !P.policy, wb);
  // exogenous inputs for this step and the obs globals of the next one, in
  // flight together with the tile copies
  const Frame F = load_frame<M>(P, E.step, E.day);
  const ObsGlobals G = load_obs_globals(P, E.step + 1, E.day);
  const uint64_t occ_ports = tile_issue_ports(P, tile, b0, lane, wb, C::stream);
  if (C::stream && P.pf_dist) {
    const int64_t bp0 = b0 + 32 * P.pf_dist;
    if (bp0 + 32 <= P.B) tile_prefetch_l2(P, bp0, lane, occ_ports, C::battery(P));
  }
  if (P.policy) policy_row(P, tile, b0, lane, pol_call);  // ALU work under the copies' latency
  tile_wait(wb);
  // state goes back to HBM port by port; obs staged in the consumed port slots,
  // or (streamed tile) through the per-port chunk ring
  const ObsSink S = C::stream ? make_chunk_sink<M>(P, T, b0, P.out.obs, /*state_to_hbm=*/true)
                              : make_sink<M>(P, T, b, P.out.obs, /*in_place=*/true);
  const int dt = P.act_dtype;
  const int64_t rs = P.act_row, cs = P.act_col;
  const uint8_t* arow = vy_smem + tile + P.L.acts + lane * (P.n_ports + 1);
  const bool staged = C::staged(P);
  auto act = [&](int slot) -> int {
    if (staged) return arow[slot];
    if (!active) return P.k;
    const int64_t at = b * rs + slot * cs;
    if (dt == VY_ACT_U8) return __ldg(reinterpret_cast<const uint8_t*>(P.actions) + at);
    if (dt == VY_ACT_I32) return __ldg(reinterpret_cast<const int32_t*>(P.actions) + at);
    const long long v = __ldg(reinterpret_cast<const long long*>(P.actions) + at);
    return v < INT_MIN ? INT_MIN : (v > INT_MAX ? INT_MAX : (int)v);
  };
  StepResult r{0.0, false};
  if (!C::probe(P, 0x200u)) r = tile_step<M>(P, prof, dtab, pc, tc, T, E, b, F, S, active, act, &occ_ports);  // 0x200: probe
  bool reset = false;
  if (r.done && (P.flags & VY_F_AUTO_RESET)) {
    // in-kernel auto-reset (engine.py:460-462): the terminal reward/done/infos
    // stand, the obs row becomes the reset obs of episode + 1
    const int ep = active ? P.st.episode[b] + 1 : 0;
    reset_scalars(P, E, active ? P.st.env_seed[b] : 0ull, ep, 0, false);
    for (int i = 0; i < P.n_ports; ++i) {
      if (active) store_port(P, b, i, 0u, 0.0, 0.0, 0.0, 0);
      if (!S.chunk) stage_port_obs(P, prof, S, lane, active, i, 0u, 0.0, 0.0, 0.0, 0, 1.0, 1.0);  // I = 0: any denominator
    }
    if (active) P.st.episode[b] = ep;
    reset = true;
  }
  if (S.chunk && (P.flags & VY_F_AUTO_RESET)) {
    // the reset obs of every env that just finished: all port columns +0
    const uint32_t dm = __ballot_sync(0xffffffffu, r.done);
    if (dm) {
      __syncwarp();  // after this step's port read-outs and arrival rows
      for (int i = 0; i < P.n_ports; ++i) chunk_zero6(S, lane, i, dm);
    }
  }
  if (active) {
    if (!C::probe(P, 0x800u)) store_env<M>(P, b, E, reset);
    if (C::f64(P))
      reinterpret_cast<double*>(P.out.reward)[b] = r.reward;
    else
      reinterpret_cast<float*>(P.out.reward)[b] = (float)r.reward;
    P.out.done[b] = r.done;
  }
  // the next tile is claimed before the obs read-out so the atomic's round
  // trip overlaps it (and not earlier: a claim held across a whole step
  // lengthens the tail of the launch)
  if (claim && lane == 0) *claim = atomicAdd(claim_ctr ? claim_ctr : P.tile_ctr, 1ull);
  emit_tail<M>(P, T, E, G, S, b0, active, P.out.obs);
}

// Persistent: one CTA per resident slot (tables staged once per CTA); each
// warp claims 32-env tiles from a global counter until none are left, so no
// warp idles waiting for the slowest warp of its CTA and the tail is balanced
// dynamically.  The last warp to finish resets the counters, which keeps the
// launch replayable inside CUDA graphs.
template <int M>
__global__ void __launch_bounds__(256) k_step(const __grid_constant__ Params P) {
  Prof prof;
  PortC pc;
  TreeC tc;
  const double* dtab;
  stage_tables(P, prof, dtab, pc, tc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t toff = tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes) + warp * P.L.bytes;
  const unsigned long long ntiles = (unsigned long long)((P.B + 31) >> 5);
  // fused RandomPolicy: the call index, from the device counter when the
  // launch is graph-replayed (advanced below by the last warp to finish, after
  // every warp has read it)
  const int64_t pol_call = P.policy ? P.pol_call + (P.pol_counter ? *(volatile int64_t*)P.pol_counter : 0) : 0;
  WarpBar wb = warp_bar_init(P, toff, lane);
  unsigned long long nxt = 0;  // lane 0: this warp's next tile (claimed inside step_tile)
  if (lane == 0) nxt = atomicAdd(P.tile_ctr, 1ull);
  for (;;) {
    const unsigned long long t = __shfl_sync(0xffffffffu, nxt, 0);
    if (t >= ntiles) break;
    step_tile<M>(P, prof, dtab, pc, tc, toff, (int64_t)t * 32, lane, wb, &nxt, pol_call);
    __syncwarp();
  }
  if (lane == 0) {
    __threadfence();  // this warp's last claim is ordered before its exit count
    const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(P.tile_ctr + 1, 1ull) == warps - 1) {
      P.tile_ctr[0] = 0;
      P.tile_ctr[1] = 0;
      if (P.policy && P.pol_counter) P.pol_counter[0] += 1;
    }
  }
}

// ---- heterogeneous batch in one launch (config C5) -------------------------
//
// Many station/market configurations ("groups", each a regular handle with
// its own tables, state and outputs) stepped by ONE persistent launch.  Global
// tile t belongs to group g with tile0[g] <= t < tile0[g+1] (the per-tile
// config index); a warp claims global tiles from one counter and steps each
// with its group's Params (stacked in global memory, read through the
// read-only path) and its group's table set (car profiles, action grid,
// per-port constants, capacity tree), every distinct set staged once per CTA
// in shared memory.  Every group's trajectory is bit-identical to stepping it
// alone: the same step_tile code runs on the same tables and state.
constexpr int kMaxGroups = 64;
// 7 warps x 2 CTAs per SM fill shared memory; the bound lets ptxas use up to 144 registers
constexpr int kMultiThreads = 224;
constexpr int kMaxSets = 8;
// Group Params live in constant memory (slot-allocated per multi handle): a
// warp-uniform group index reads them through the constant cache into
// uniform registers, like a single launch's __grid_constant__ Params (a
// global-memory copy measured 10-20% slower: loads in the dependency chains
// and per-thread registers for every hoisted field).
constexpr int kConstGroups = 48;  // 48 x 1136 B of the 64 KB constant bank
__constant__ Params c_groups[kConstGroups];

struct MultiArgs {
  int slot0;                // first c_groups slot of this batch
  int n_groups, n_psets, n_ssets;
  int64_t tile0[kMaxGroups + 1];  // first global tile of each group; tile0[n_groups] = total
  int8_t group_pset[kMaxGroups];  // car-profile set of each group
  int8_t group_sset[kMaxGroups];  // station set (action grid, per-port constants, tree) of each group
  int pset_group[kMaxSets], sset_group[kMaxSets];  // a group whose tables define the set
  int pset_off[kMaxSets], sset_off[kMaxSets];      // smem byte offsets of the staged sets
  int tiles_off;                  // smem byte offset of warp tile 0
  int tile_bytes;                 // bytes per warp tile (max over groups)
  unsigned long long* ctr;        // [2] tile counter, finished warps
  int64_t pol_call;               // RandomPolicy call index (+ *pol_counter when set)
  int64_t* pol_counter;
};
// station set layout: action grid (2k+1 doubles, 16-aligned), per-port constants, tree
__host__ __device__ inline int sset_portc_off(int k) { return ((2 * k + 1) * 8 + 15) & ~15; }
__host__ __device__ inline int sset_treec_off(int k, int n_ports) { return sset_portc_off(k) + n_ports * 8 * kPortWords; }
__host__ __device__ inline int sset_bytes(int k, int n_ports, int n_nodes) {
  return (sset_treec_off(k, n_ports) + n_nodes * 32 + 15) & ~15;
}
__host__ __device__ inline int pset_bytes(int n_profiles) { return (n_profiles * (int)sizeof(Profile) + 15) & ~15; }

__device__ __forceinline__ void stage_multi_sets(const MultiArgs& A) {
  for (int s = 0; s < A.n_psets; ++s) {
    const Params& P = c_groups[A.slot0 + A.pset_group[s]];
    double* d = reinterpret_cast<double*>(vy_smem + A.pset_off[s]);
    const double* gp = reinterpret_cast<const double*>(P.profiles);
    for (int i = threadIdx.x; i < P.n_profiles * kProfileWords; i += blockDim.x) d[i] = __ldg(gp + i);
  }
  for (int s = 0; s < A.n_ssets; ++s) {
    const Params& P = c_groups[A.slot0 + A.sset_group[s]];
    unsigned char* base = vy_smem + A.sset_off[s];
    double* sd = reinterpret_cast<double*>(base);
    for (int i = threadIdx.x; i < 2 * P.k + 1; i += blockDim.x) sd[i] = __ldg(P.delta_tab + i);
    double* sp = reinterpret_cast<double*>(base + sset_portc_off(P.k));
    for (int i = threadIdx.x; i < P.n_ports * kPortWords; i += blockDim.x) sp[i] = __ldg(P.portc + i);
    double* st = reinterpret_cast<double*>(base + sset_treec_off(P.k, P.n_ports));
    for (int i = threadIdx.x; i < P.n_nodes * 4; i += blockDim.x) st[i] = __ldg(P.treec + i);
  }
}

template <int M>
__global__ void __launch_bounds__(kMultiThreads) k_step_multi(const __grid_constant__ MultiArgs A) {
  stage_multi_sets(A);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t toff = (uint32_t)(A.tiles_off + warp * A.tile_bytes);
  WarpBar wb{smem_base() + toff + (uint32_t)A.tile_bytes - 16u, 0u, false};
  if (lane == 0) {
    mbar_init(wb.a);
    mbar_init_fence();
  }
  __syncwarp();
  const unsigned long long ntiles = (unsigned long long)A.tile0[A.n_groups];
  const int64_t pol_call = A.pol_call + (A.pol_counter ? *(volatile int64_t*)A.pol_counter : 0);
  unsigned long long nxt = 0;
  if (lane == 0) nxt = atomicAdd(A.ctr, 1ull);
  for (;;) {
    const unsigned long long t = __shfl_sync(0xffffffffu, nxt, 0);
    if (t >= ntiles) break;
    // group: last g with tile0[g] <= t, from two warp votes over the tile
    // offsets (a vote result is warp-uniform, so the group's Params below are
    // read with uniform constant loads into uniform registers)
    const unsigned v0 = __ballot_sync(0xffffffffu, lane < A.n_groups && (unsigned long long)A.tile0[lane] <= t);
    const unsigned v1 =
        __ballot_sync(0xffffffffu, lane + 32 < A.n_groups && (unsigned long long)A.tile0[lane + 32] <= t);
    const int g = __popc(v0) + __popc(v1) - 1;
    const Params& P = c_groups[A.slot0 + g];
    const uint32_t so = (uint32_t)A.sset_off[A.group_sset[g]];
    const int kk = P.k;
    const Prof prof{smem_base() + (uint32_t)A.pset_off[A.group_pset[g]]};
    const PortC pc{smem_base() + so + (uint32_t)sset_portc_off(kk)};
    const TreeC tc{smem_base() + so + (uint32_t)sset_treec_off(kk, P.n_ports)};
    const double* dtab = reinterpret_cast<const double*>(vy_smem + so);
    step_tile<M>(P, prof, dtab, pc, tc, toff, ((int64_t)t - A.tile0[g]) * 32, lane, wb, &nxt, pol_call, A.ctr);
    __syncwarp();
  }
  if (lane == 0) {
    __threadfence();
    const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(A.ctr + 1, 1ull) == warps - 1) {
      A.ctr[0] = 0;
      A.ctr[1] = 0;
      if (A.pol_counter) A.pol_counter[0] += 1;
    }
  }
}

#ifndef VY_ROLL_U2
#define VY_ROLL_U2 2  // the rollout's charge/departure loop unroll (tile_step U2)
#endif
template <int M>
__global__ void __launch_bounds__(256) k_rollout(const __grid_constant__ Params P, int T_steps, uint64_t policy_seed,
                                                 int64_t index0, int64_t call0, int64_t obs_stride,
                                                 int64_t rew_stride) {
  using C = Spec<M>;
  Prof prof;
  PortC pc;
  TreeC tc;
  const double* dtab;
  stage_tables(P, prof, dtab, pc, tc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32;
  if (b0 >= P.B) return;
  const uint32_t tile = tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes) + warp * P.L.bytes;
  const Lane T = make_lane(P, tile, lane);
  const int64_t b = b0 + lane;
  const bool active = b < P.B;
  WarpBar wb = warp_bar_init(P, tile, lane);
  tile_issue(P, tile, b0, lane, false, wb);
  tile_wait(wb);
  EnvRegs E{};  // zero for padding lanes so the obs path stays in bounds
  uint64_t pkey = 0, seed = 0;
  int episode = 0;
  if (active) {
    load_env<M>(P, b, E);
    pkey = fold(fold(fold(kKey0, policy_seed), (uint64_t)(index0 + b)), 2);
    episode = P.st.episode[b];
    seed = P.st.env_seed[b];
  }
  const int ns = P.n_ports + 1, hi = 2 * P.k + 1;
  const bool f64 = C::f64(P);
  for (int t = 0; t < T_steps; ++t) {
    void* obs_t = f64 ? (void*)(reinterpret_cast<double*>(P.out.obs) + t * obs_stride)
                      : (void*)(reinterpret_cast<float*>(P.out.obs) + t * obs_stride);
    const ObsSink S = make_chunk_sink<M>(P, T, b0, obs_t);
    const uint64_t j0 = (uint64_t)(call0 + t) * (uint64_t)ns;
    auto act = [&](int slot) -> int { return policy_action(pkey, j0 + slot + 1, hi); };
    const Frame F = load_frame<M>(P, E.step, E.day);
    const StepResult r = tile_step<M, decltype(act), VY_ROLL_U2>(P, prof, dtab, pc, tc, T, E, b, F, S, active, act, nullptr);
    if (r.done) {
      ++episode;
      reset_scalars(P, E, seed, episode, 0, false);
      clear_tile_ports(P, T);
      if (!S.chunk)
        for (int i = 0; i < P.n_ports; ++i) stage_port_obs(P, prof, S, lane, active, i, 0u, 0.0, 0.0, 0.0, 0, 1.0, 1.0);
    }
    if (S.chunk) {
      // the reset obs of every env that just finished: all port columns +0
      const uint32_t dm = __ballot_sync(0xffffffffu, r.done);
      if (dm) {
        __syncwarp();  // after this step's port read-outs and arrival rows
        for (int i = 0; i < P.n_ports; ++i) chunk_zero6(S, lane, i, dm);
      }
    }
    if (active) {
      if (f64)
        reinterpret_cast<double*>(P.out.reward)[t * rew_stride + b] = r.reward;
      else
        reinterpret_cast<float*>(P.out.reward)[t * rew_stride + b] = (float)r.reward;
      P.out.done[t * rew_stride + b] = r.done;
    }
    emit_tail<M>(P, T, E, load_obs_globals(P, E.step, E.day), S, b0, active, obs_t);
  }
  if (!C::probe(P, 0x800u)) tile_store(P, T.t, b0, lane);
  if (active) {
    store_env<M>(P, b, E, true);
    P.st.episode[b] = episode;
  }
}

__global__ void __launch_bounds__(256) k_reset(const __grid_constant__ Params P, const uint8_t* mask,
                                               int episode_mode, const int32_t* inj_day,
                                               const int32_t* episodes) {
  Prof prof;
  PortC pc;
  TreeC tc;
  const double* dtab;
  stage_tables(P, prof, dtab, pc, tc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32;
  if (b0 >= P.B) return;
  const uint32_t tile = tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes) + warp * P.L.bytes;
  const Lane T = make_lane(P, tile, lane);
  const int64_t b = b0 + lane;
  const bool active = b < P.B;
  // masked-out envs keep their state: stage the tile so the write-back is a no-op for them
  WarpBar wb = warp_bar_init(P, tile, lane);
  tile_issue(P, tile, b0, lane, false, wb);
  tile_wait(wb);
  const bool mine = active && (!mask || mask[b]);
  EnvRegs E{};  // zero for padding lanes so the obs path stays in bounds
  if (active) load_env<0>(P, b, E);
  if (mine) {
    const int ep = episodes ? episodes[b] : (episode_mode ? P.st.episode[b] + 1 : 0);
    reset_scalars(P, E, P.st.env_seed[b], ep, inj_day ? inj_day[b] : 0, inj_day != nullptr);
    clear_tile_ports(P, T);
    P.st.episode[b] = ep;
    store_env<0>(P, b, E, true);
  }
  // masked-out rows still get their (unchanged) obs rewritten, which is idempotent
  emit_obs(P, prof, pc, T, E, load_obs_globals(P, E.step, E.day), b0, active, P.out.obs, /*store_state=*/true);
}

}  // namespace vy
