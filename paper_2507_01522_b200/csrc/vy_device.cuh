// vy_device.cuh — launch parameters, per-warp tile layout, and the
// splitmix64 stream on the device.
//
// The RNG is the reference's own counter-based stream (rng.py:20-115,
// _kernel.pyx:19-73): draw j of key k is mix64(k + j*GOLDEN).  Being
// counter-based, every env regenerates exactly the reference's draws with no
// sequential host state, so arrivals and the reset day are bit-identical to
// the CPU reference at any batch size.  An injected draw buffer (vy_draws)
// can replace the arrival draws (VY_F_INJECT).
#pragma once

#include <cstdint>

#include "../../include/voltyard_b200.h"

namespace vy {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kKey0 = 0x8C2F9D1B6E4A5533ULL;
constexpr int kMaxPorts = 64;
constexpr int kMaxNodes = 2 * kMaxPorts + 2;
constexpr int kMaxProfiles = 64;  // 6 bits of port_meta
constexpr int kFastNodes = 4;     // trees up to this many nodes keep node loads in registers
// per-port constant record (PortC in vy_tile.cuh), 16-byte pairs in the order the step uses them:
// {imax_c, imax_d} {volt, rcp_volt} {kind, node mask} {dtv, eta_d} {eta_c, rcp_eta_c} {i_denom, rcp_i_denom}
constexpr int kPortWords = 12;
constexpr uint32_t kFlagStageObs = 0x100u;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t fold(uint64_t key, uint64_t part) { return mix64((key + kGolden) ^ part); }
// uniform in [0,1) with 53 random bits; exact conversion, exact scaling
__device__ __forceinline__ double unit(uint64_t& st) {
  st += kGolden;
  return __dmul_rn((double)(mix64(st) >> 11), 1.0 / 9007199254740992.0);
}
__device__ __forceinline__ int below(uint64_t& st, int n) {  // Stream.randint
  const int k = (int)__double2ll_rz(__dmul_rn(unit(st), (double)n));
  return k >= n ? n - 1 : k;
}
// Knuth product of uniforms against a host-computed exp(-lambda) threshold
__device__ __forceinline__ int knuth(uint64_t& st, double thr) {
  double p = 1.0;
  int k = 0;
  for (;;) {
    p = __dmul_rn(p, unit(st));
    if (p <= thr) return k;
    ++k;
  }
}
// RandomPolicy draw: row key k, overall draw number j (1-based), hi = 2K+1.
// The reference's u * hi with u = m * 2^-53 (m = x >> 11, exact) is the single
// rounding RN(m * hi * 2^-53) = RN(m * (hi * 2^-53)): one multiply by the
// exact constant hi * 2^-53.
__device__ __forceinline__ int policy_action(uint64_t key, uint64_t j, int hi) {
  const double uh = __dmul_rn((double)(mix64(key + j * kGolden) >> 11), (double)hi * (1.0 / 9007199254740992.0));
  const int a = (int)__double2int_rz(uh);
  return a >= hi ? hi - 1 : a;
}

// x / d for a divisor d > 0 known ahead of time, with y = RN(1/d) precomputed:
// q = RN(x*y) is within 1 ulp of x/d, r = x - q*d is exact (FMA), and
// RN(q + r*y) is the correctly rounded quotient (Markstein's theorem for a
// correctly rounded reciprocal; no under/overflow in this model's ranges).
// Bit-identical to IEEE x / d, checked exhaustively-by-sampling by
// vy_selftest_div (tests/test_gpu_numerics.py).  The residual is formed as
// -(q*d - x) rather than x - q*d: the same exact value, but a zero dividend
// yields a -0 residual, so RN(q + (-0)*y) keeps the sign of a zero quotient
// with no select or branch (three fp64 instructions in all).
__device__ __forceinline__ double div_rcp(double x, double d, double y) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(q, d, -x);
  return __fma_rn(-r, y, q);
}

struct Profile {  // car profile: catalogue entry (or injected car)
  double cap, r_ac, r_dc, tau, omt;  // omt = 1.0 - tau, same rounding as the reference's runtime expression
  double rcp_cap, rcp_omt;           // RN(1/cap), RN(1/omt)
  double cum;     // catalogue entries: cumulative sampling weight (data.py:112-114), read by the arrivals' car draw
  double pad;     // 72-byte stride: profiles 0..4 start in distinct bank pairs (per-lane lookups of different cars)
};

// Byte offsets inside one warp's shared-memory tile (32 envs, lane = env).
// Per-port fields are [port][lane]; per-env fields [lane].  The float64 port
// slots (idr/soc/de, 256 B per port each) are reused as the obs staging area
// once a port has been written back.
//   [pad 24n][port][idr, soc, de][lane] f64 (n x 768 B at `ports`),
//   dwell [port][lane] i16, meta [port][lane] u8, actions [lane][n+1] u8.
//   Obs staging: column c, row r at obs + c*132 + r*4 (33-word columns: per
//   lane writes and per row reads are both bank-conflict free).  In the step
//   kernel obs = 0: column block 6i..6i+5 (792 B) fits in front of port i+1's
//   slots thanks to the 24n-byte pad, so the staging reuses the consumed port
//   slots; rollouts keep their state and stage in a separate area.
struct TileLayout {
  int ports;  // byte offset of port 0's float64 slots (port i at ports + i*768)
  int dtrem, meta, acts;
  int obs;    // byte offset of obs column 0 (0 in-place; `extra` area for rollouts)
  int bar;    // byte offset of the warp's mbarrier (8 B) completing the tile's bulk copies
  int ps;     // bytes between consecutive ports' slots: 768 (i_drawn, soc, de) or 256 (streamed tile: i_drawn)
  int bytes;
};

struct Params {
  // shape
  int n_ports, n_slots, n_nodes, max_passes;
  int k, episode_steps, steps_per_day, dt_min, horizon, obs_len, n_days, lam_len, n_cat;
  int stay_lo, stay_span, allow_discharge, battery, has_moer, has_dgrid, order_identity;
  int64_t B, ld;
  uint32_t flags;
  double dt_h, p_sell, c_dt, beta, soc_lo, soc_span, frac_lo, frac_span, p_charge, thr32;
  double alphas[8];
  // battery
  double b_volt, b_cap, b_rmax, b_tau, b_omt, b_eta_c, b_eta_d, b_init_soc, b_imax, b_idenom, b_dtv;
  double b_rcp_volt, b_rcp_cap, b_rcp_omt, b_rcp_eta_c, b_rcp_idenom;
  double rcp_1000, rcp_ep, rcp_365;
  int battery_node_mask;  // bit m: battery slot in node m's range (m < kFastNodes)
  int act_tile;           // actions are row-major uint8 [B][n+1], staged per tile
  int n_profiles;         // live entries of the car-profile table
  // ports: per-port constants live in `portc` (staged per CTA); the parking
  // order (generic path only) in device memory
  const int* order;  // [n_ports]
  // capacity tree: the fast (register) path's nodes m < kFastNodes; every node in `treec`
  double node_cap[kFastNodes], node_eta[kFastNodes], node_rcp_eta[kFastNodes];
  // series (device)
  const double *buy, *sellg, *moer, *dgrid, *sin_t, *cos_t, *cat_cum;
  const int8_t* weekday;
  const double* pois_thr;   // [2][lam_len] threshold of the last (partial) chunk
  const int* pois_full;     // [2][lam_len] number of full 32-chunks; -1 => lambda <= 0
  const Profile* profiles;  // [kMaxProfiles]
  const double* delta_tab;  // [2k+1] (a-k)/k
  const double* portc;      // [n_ports][kPortWords] per-port constants, staged into shared memory (PortC)
  const double* treec;      // [n_nodes][4] tree nodes in deepest-first order, staged into shared memory (TreeC)
  // state / outputs / actions
  vy_state st;
  vy_outputs out;
  const void* actions;
  int act_dtype;
  int64_t act_row, act_col;
  vy_draws inj;
  // fused RandomPolicy (vy_step_random): actions generated in the step kernel
  int policy;                 // 1: actions are RandomPolicy draws, not read from `actions`
  uint64_t pol_seed;
  int64_t pol_index0, pol_call;
  int64_t* pol_counter;       // {call index, finished warps}: device call counter (graph replay), or null
  uint8_t* pol_out;           // optional uint8 [B][n+1] copy of the generated actions
  uint32_t* err;
  unsigned long long* tile_ctr;  // [2] work-stealing tile counter, finished-warp counter (k_step)
  int64_t pf_dist;               // streamed k_step: L2 prefetch of tile t + pf_dist while tile t runs (0: off)
  TileLayout L;
};


// Compile-time specialisation.  Spec<M>, M = 1 ("lean") is the step of the
// common configuration: obs/reward/done only (no infos, no injected draws),
// float32 obs, no battery, no carbon / demand series, no price horizon, a
// tree of at most kFastNodes nodes, identity parking order, staged uint8
// actions, a shuffle-sized action grid.  M = 2 is the same with a larger tree
// (node loads summed from the tile, vy_tile.cuh node_sum); M = 3 adds the
// stationary battery (any tree) — the config-C4 station.  Everything a lean
// mode folds away is dead code its kernel never carries (smaller hot loop,
// fewer i-cache misses, no uniform branches); M = 0 reads all of it at run
// time.  The host picks the instantiation (step_mode in vy_abi.cu).
template <int M>
struct Spec {
  static constexpr bool lean = M != 0;
  __device__ __forceinline__ static bool info(const Params& P) { return !lean && (P.flags & VY_F_INFOS); }
  __device__ __forceinline__ static bool inject(const Params& P) { return !lean && (P.flags & VY_F_INJECT); }
  __device__ __forceinline__ static bool f64(const Params& P) { return !lean && (P.flags & VY_F_OUT_F64); }
  // M = 4: M = 3 with a streamed tile (large battery stations, e.g. config C4):
  // only the port currents stay in shared memory; soc / energy / dwell are
  // read from HBM a few ports ahead in the port loops, obs leave through the
  // per-port chunk ring, so a 64-port tile needs ~22 KB instead of ~62 KB
  static constexpr bool stream = M == 4;
  __device__ __forceinline__ static bool battery(const Params& P) { return (M == 0 || M == 3 || M == 4) && P.battery; }
  __device__ __forceinline__ static bool moer(const Params& P) { return !lean && P.has_moer; }
  __device__ __forceinline__ static bool dgrid(const Params& P) { return !lean && P.has_dgrid; }
  __device__ __forceinline__ static int horizon(const Params& P) { return lean ? 0 : P.horizon; }
  __device__ __forceinline__ static bool fast_tree(const Params& P) {
    return M == 1 || ((M == 0 || M == 3 || M == 4) && P.n_nodes <= kFastNodes);
  }
  __device__ __forceinline__ static bool identity(const Params& P) { return lean || P.order_identity; }
  __device__ __forceinline__ static bool staged(const Params& P) { return lean || P.act_tile; }
  __device__ __forceinline__ static bool probe(const Params& P, uint32_t bit) { return !lean && (P.flags & bit); }
};

}  // namespace vy
