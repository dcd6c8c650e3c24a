// vy_device.cuh — launch parameters and the splitmix64 stream on the device.
//
// The RNG is the reference's own counter-based stream (rng.py:20-115,
// _kernel.pyx:19-73): draw j of key k is mix64(k + j*GOLDEN).  Being
// counter-based, every env regenerates exactly the reference's draws with no
// sequential host state, so arrivals and the reset day are bit-identical to
// the CPU reference at any batch size ("reference stream" mode).  An injected
// draw buffer (vy_draws) can replace the arrival draws (VY_F_INJECT).
#pragma once

#include <cstdint>

#include "../../include/voltyard_b200.h"

namespace vy {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kKey0 = 0x8C2F9D1B6E4A5533ULL;
constexpr int kMaxProfiles = 64;  // 6 bits of port_meta

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
  int k = (int)__double2ll_rz(__dmul_rn(unit(st), (double)n));
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

struct Profile {  // car profile: catalogue entry (or injected car)
  double cap, r_ac, r_dc, tau, omt;  // omt = 1.0 - tau, same rounding as the reference's runtime expression
};

// Everything a launch reads besides state: scalars by value (constant bank),
// per-port / per-node arrays sized by the template port capacity NP, and
// device pointers to the long series.
template <int NP>
struct Params {
  static constexpr int NS = NP + 1;
  static constexpr int NN = 2 * NP + 2;  // node capacity
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
  // ports (index = compile-time port number)
  double volt[NP], imax_c[NP], imax_d[NP], eta_c[NP], eta_d[NP], i_denom[NP], dtv[NP];
  int kind[NP], order[NP];
  // capacity tree: node m sums slots [lo, hi) in order
  double node_cap[NN], node_eta[NN];
  int node_lo[NN], node_hi[NN], node_order[NN];
  // series (device)
  const double *buy, *sellg, *moer, *dgrid, *sin_t, *cos_t, *cat_cum;
  const int8_t* weekday;
  const double* pois_thr;   // [2][lam_len] threshold of the last (partial) chunk
  const int* pois_full;     // [2][lam_len] number of full 32-chunks; -1 => lambda <= 0
  const Profile* profiles;  // [kMaxProfiles]
  const double* delta_tab;  // [2k+1] (a-k)/k
  // state / outputs / actions
  vy_state st;
  vy_outputs out;
  const void* actions;
  int act_dtype;
  int64_t act_row, act_col;
  vy_draws inj;
  uint32_t* err;
};

}  // namespace vy
