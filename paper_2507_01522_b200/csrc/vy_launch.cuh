// vy_launch.cuh — handle layout and per-port-capacity launchers.  Each
// capacity NP is instantiated in its own translation unit (vy_np*.cu) so the
// register-heavy kernels compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "vy_kernels.cuh"

namespace vy {
int fail(int code, const std::string& msg);
}  // namespace vy

#define VY_CUDA(call)                                                                                  \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) return ::vy::fail(VY_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

struct vy_handle {
  using Profile = vy::Profile;
  int device = 0;
  int64_t B = 0;
  int np = 0;
  vy_tables t{};  // scalars only (pointers are not retained)
  std::vector<double> volt, imax_c, imax_d, eta_c, eta_d, i_denom, node_cap, node_eta;
  std::vector<int> kind, order, node_lo, node_hi, node_order;
  bool order_identity = true;
  std::vector<Profile> profiles;
  double *d_buy = nullptr, *d_sellg = nullptr, *d_moer = nullptr, *d_dgrid = nullptr, *d_sin = nullptr,
         *d_cos = nullptr, *d_catcum = nullptr, *d_pthr = nullptr, *d_dtab = nullptr;
  int8_t* d_wk = nullptr;
  int* d_pfull = nullptr;
  Profile* d_prof = nullptr;
  uint32_t* d_err = nullptr;
  double thr32 = 0.0;
  vy_state st{};
  vy_outputs out{};
  bool bound = false;
  int64_t launches = 0;
  size_t smem_limit = 0;
};


namespace vy {

template <int NP>
int launch_step(vy_handle* h, const void* actions, int dtype, int64_t rs, int64_t cs, uint32_t flags,
                const vy_draws* inj, cudaStream_t s);
template <int NP>
int launch_reset(vy_handle* h, const uint8_t* mask, int mode, const int32_t* inj_day, uint32_t flags,
                 cudaStream_t s);
template <int NP>
int launch_rollout(vy_handle* h, int T, uint64_t seed, int64_t index0, int64_t call0, void* obs, int64_t obs_stride,
                   void* reward, uint8_t* done, int64_t rew_stride, uint32_t flags, cudaStream_t s);

#ifdef VY_DEFINE_LAUNCHERS
template <int NP>
int fill(vy_handle* h, Params<NP>& P) {
  const vy_tables& t = h->t;
  std::memset(&P, 0, sizeof(P));
  P.n_ports = t.n_ports;
  P.n_slots = t.n_slots;
  P.n_nodes = t.n_nodes;
  P.max_passes = t.max_passes;
  P.k = t.k;
  P.episode_steps = t.episode_steps;
  P.steps_per_day = t.steps_per_day;
  P.dt_min = t.dt_min;
  P.horizon = t.horizon;
  P.obs_len = t.obs_len;
  P.n_days = t.n_days;
  P.lam_len = t.lam_len;
  P.n_cat = t.n_cat;
  P.stay_lo = t.stay_lo;
  P.stay_span = t.stay_hi - t.stay_lo + 1;
  P.allow_discharge = t.allow_discharge;
  P.battery = t.battery_enabled;
  P.has_moer = t.has_moer;
  P.has_dgrid = t.has_dgrid;
  P.order_identity = h->order_identity;
  P.B = h->B;
  P.ld = h->st.ld;
  P.dt_h = t.dt_h;
  P.p_sell = t.p_sell;
  P.c_dt = t.c_dt;
  P.beta = t.beta;
  P.soc_lo = t.soc_lo;
  P.soc_span = t.soc_hi - t.soc_lo;  // same runtime expression as _kernel.pyx:486
  P.frac_lo = t.frac_lo;
  P.frac_span = t.frac_hi - t.frac_lo;
  P.p_charge = t.p_charge;
  P.thr32 = h->thr32;
  for (int i = 0; i < 8; ++i) P.alphas[i] = t.alphas[i];
  P.b_volt = t.b_volt;
  P.b_cap = t.b_cap;
  P.b_rmax = t.b_rmax;
  P.b_tau = t.b_tau;
  P.b_omt = 1.0 - t.b_tau;
  P.b_eta_c = t.b_eta_c;
  P.b_eta_d = t.b_eta_d;
  P.b_init_soc = t.b_init_soc;
  P.b_imax = t.b_imax;
  P.b_idenom = t.b_idenom;
  P.b_dtv = t.dt_h * t.b_volt;
  for (int i = 0; i < t.n_ports; ++i) {
    P.volt[i] = h->volt[i];
    P.imax_c[i] = h->imax_c[i];
    P.imax_d[i] = h->imax_d[i];
    P.eta_c[i] = h->eta_c[i];
    P.eta_d[i] = h->eta_d[i];
    P.i_denom[i] = h->i_denom[i];
    P.dtv[i] = t.dt_h * h->volt[i];  // (dt_h * V) * I / 1000 evaluates left to right (_kernel.pyx:366)
    P.kind[i] = h->kind[i];
    P.order[i] = h->order[i];
  }
  for (int m = 0; m < t.n_nodes; ++m) {
    P.node_cap[m] = h->node_cap[m];
    P.node_eta[m] = h->node_eta[m];
    P.node_lo[m] = h->node_lo[m];
    P.node_hi[m] = h->node_hi[m];
    P.node_order[m] = h->node_order[m];
  }
  P.buy = h->d_buy;
  P.sellg = h->d_sellg;
  P.moer = h->d_moer;
  P.dgrid = h->d_dgrid;
  P.sin_t = h->d_sin;
  P.cos_t = h->d_cos;
  P.cat_cum = h->d_catcum;
  P.weekday = h->d_wk;
  P.pois_thr = h->d_pthr;
  P.pois_full = h->d_pfull;
  P.profiles = h->d_prof;
  P.delta_tab = h->d_dtab;
  P.st = h->st;
  P.out = h->out;
  P.err = h->d_err;
  return VY_OK;
}

template <typename K>
inline int ensure_smem(K kernel, int bytes) {
  if (bytes > 48 * 1024) VY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return VY_OK;
}

inline bool can_stage(vy_handle* h, uint32_t flags, const void* obs) {
  if (flags & VY_F_OUT_F64) return false;
  if (reinterpret_cast<uintptr_t>(obs) % 16) return false;
  const SmemLayout L = smem_layout(h->t.k, h->t.obs_len, true);
  return L.bytes <= 160 * 1024;
}

template <int NP>
int launch_step(vy_handle* h, const void* actions, int dtype, int64_t rs, int64_t cs, uint32_t flags,
                const vy_draws* inj, cudaStream_t s) {
  Params<NP> P;  // built on the host, passed by value
  fill<NP>(h, P);
  const bool stage = can_stage(h, flags, h->out.obs);
  P.flags = flags | (stage ? 0x100u : 0u);
  P.actions = actions;
  P.act_dtype = dtype;
  P.act_row = rs;
  P.act_col = cs;
  if (inj) P.inj = *inj;
  const SmemLayout L = smem_layout(h->t.k, h->t.obs_len, stage);
  if (ensure_smem(k_step<NP>, L.bytes)) return VY_ERR_CUDA;
  const unsigned grid = (unsigned)((h->B + kBlock - 1) / kBlock);
  k_step<NP><<<grid, kBlock, L.bytes, s>>>(P);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

template <int NP>
int launch_reset(vy_handle* h, const uint8_t* mask, int mode, const int32_t* inj_day, uint32_t flags,
                 cudaStream_t s) {
  Params<NP> P;
  fill<NP>(h, P);
  P.flags = flags;
  const SmemLayout L = smem_layout(h->t.k, h->t.obs_len, false);
  if (ensure_smem(k_reset<NP>, L.bytes)) return VY_ERR_CUDA;
  const unsigned grid = (unsigned)((h->B + kBlock - 1) / kBlock);
  k_reset<NP><<<grid, kBlock, L.bytes, s>>>(P, mask, mode, inj_day);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

template <int NP>
int launch_rollout(vy_handle* h, int T, uint64_t seed, int64_t index0, int64_t call0, void* obs, int64_t obs_stride,
                   void* reward, uint8_t* done, int64_t rew_stride, uint32_t flags, cudaStream_t s) {
  Params<NP> P;
  fill<NP>(h, P);
  const bool stage = can_stage(h, flags, obs) && (obs_stride * 4) % 16 == 0;
  P.flags = flags | (stage ? 0x100u : 0u);
  P.out.obs = obs;
  P.out.reward = reward;
  P.out.done = done;
  const SmemLayout L = smem_layout(h->t.k, h->t.obs_len, stage);
  if (ensure_smem(k_rollout<NP>, L.bytes)) return VY_ERR_CUDA;
  const unsigned grid = (unsigned)((h->B + kBlock - 1) / kBlock);
  k_rollout<NP><<<grid, kBlock, L.bytes, s>>>(P, T, seed, index0, call0, obs_stride, rew_stride);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}


#define VY_INSTANTIATE(NP)                                                                                    \
  template int launch_step<NP>(vy_handle*, const void*, int, int64_t, int64_t, uint32_t, const vy_draws*,     \
                               cudaStream_t);                                                                 \
  template int launch_reset<NP>(vy_handle*, const uint8_t*, int, const int32_t*, uint32_t, cudaStream_t);     \
  template int launch_rollout<NP>(vy_handle*, int, uint64_t, int64_t, int64_t, void*, int64_t, void*, uint8_t*, \
                                  int64_t, uint32_t, cudaStream_t);
#endif

}  // namespace vy
