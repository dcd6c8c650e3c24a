// vy_abi.cu — C ABI (include/voltyard_b200.h) over the sm_100a kernels.
//
// Host responsibilities: validate and flatten the reference tables into the
// launch parameters (per-port constants by value, long series in device
// memory), precompute the values whose host computation must match the
// reference bit for bit (Poisson thresholds exp(-lambda) with the same libm
// the reference calls, _kernel.pyx:56; the (a-k)/k action grid,
// _kernel.pyx:305), size the per-warp shared-memory tiles, and launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "vy_kernels.cuh"
#include "vy_wide.cuh"
#include "vy_ppo_rollout.cuh"

using namespace vy;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define VY_CUDA(call)                                                                                       \
  do {                                                                                                      \
    cudaError_t e_ = (call);                                                                                \
    if (e_ != cudaSuccess) return fail(VY_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_));       \
  } while (0)

template <typename T>
int upload(T** dst, const T* src, size_t n) {
  if (n == 0) n = 1;
  VY_CUDA(cudaMalloc(dst, n * sizeof(T)));
  if (src) VY_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return VY_OK;
}
}  // namespace

namespace vy {

// RandomPolicy rows: thread per env computes its n+1 actions into a per-warp
// smem row block, then the warp writes the contiguous [32][n+1] byte block
// with coalesced stores (per-thread 17-byte rows would be strided byte stores).
// Device-counter mode (call_dev = {call, blocks done}): every block reads the
// call index at its start; the last block to finish advances it (and clears
// the done count), so one launch per step is graph-replayable.
__device__ __forceinline__ void bump_call(int64_t* call_dev) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    auto* done = reinterpret_cast<unsigned long long*>(call_dev + 1);
    if (atomicAdd(done, 1ull) == (unsigned long long)gridDim.x - 1) {
      call_dev[0] += 1;
      *done = 0;
    }
  }
}

__global__ void k_random_actions(uint64_t seed, int64_t index0, int64_t call, int64_t B, int ns, int hi,
                                 uint8_t* out, int64_t* call_dev) {
  if (call_dev) call += *(volatile int64_t*)call_dev;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32;
  if (b0 >= B) {  // (warp 0 of every block is in range: grid = ceil(B / block))
    if (call_dev) bump_call(call_dev);
    return;
  }
  unsigned char* rows = vy_smem + warp * 32 * ns;
  const int64_t b = b0 + lane;
  if (b < B) {
    const uint64_t key = fold(fold(fold(kKey0, seed), (uint64_t)(index0 + b)), 2);
    // draw j = call*ns + s + 1 of the row's stream is mix64(key + j*GOLDEN): step the argument by GOLDEN
    uint64_t kj = key + ((uint64_t)call * (uint64_t)ns + 1) * kGolden;
    for (int s = 0; s < ns; ++s, kj += kGolden) rows[lane * ns + s] = (uint8_t)policy_action(kj, 0, hi);
  }
  __syncwarp();
  const int64_t left = B - b0;
  const int bytes = (left >= 32 ? 32 : (int)left) * ns;
  uint8_t* g = out + b0 * ns;
  if ((bytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(rows)) & 15) == 0) {
    // a full 32-row tile is 32*ns bytes, a multiple of 16: 16-byte stores
    for (int o = lane * 16; o < bytes; o += 512)
      *reinterpret_cast<uint4*>(g + o) = *reinterpret_cast<const uint4*>(rows + o);
  } else {
    for (int o = lane; o < bytes; o += 32) g[o] = rows[o];
  }
  if (call_dev) bump_call(call_dev);
}

// div_rcp vs IEEE division on random dividends spread over 2^-64..2^64
__global__ void k_selftest_div(const double* d, const double* y, int nd, int64_t per, uint64_t seed,
                               unsigned long long* bad) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (int64_t s = gid; s < per * nd; s += stride) {
    const int k = (int)(s % nd);
    const uint64_t bits = mix64(seed + (uint64_t)s * kGolden);
    const uint64_t mant = bits & 0xFFFFFFFFFFFFFull;
    const uint64_t ex = 1023 - 64 + ((bits >> 52) & 127);  // exponents 2^-64 .. 2^63
    const uint64_t sign = bits & 0x8000000000000000ull;
    double x = __longlong_as_double((long long)(sign | (ex << 52) | mant));
    // the first 64 dividends of every divisor are the special ones the model
    // produces: signed zeros, small integers (dwell / episode_steps), exact
    // multiples and halves
    const int64_t j = s / nd;
    if (j < 64) {
      if (j < 2) x = j == 0 ? 0.0 : -0.0;
      else if (j < 34) x = (double)(j - 17);
      else if (j < 50) x = d[k] * (double)(j - 41);
      else x = 0.5 * (double)(j - 56);
    }
    const double want = __ddiv_rn(x, d[k]);
    const double got = div_rcp(x, d[k], y[k]);
    if (__double_as_longlong(want) != __double_as_longlong(got)) ++local;
  }
  if (local) atomicAdd(bad, local);
}


__global__ void k_seed_envs(uint64_t master, int64_t index0, int64_t B, uint64_t* env_seed) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) env_seed[b] = fold(fold(kKey0, master), (uint64_t)(index0 + b));
}

}  // namespace vy

struct vy_handle {
  int device = 0;
  int64_t B = 0;
  vy_tables t{};  // scalars only (pointers are not retained)
  std::vector<double> volt, imax_c, imax_d, eta_c, eta_d, i_denom, node_cap, node_eta;
  std::vector<int> kind, order, node_lo, node_hi, node_order;
  bool order_identity = true;
  std::vector<Profile> profiles;
  double *d_buy = nullptr, *d_sellg = nullptr, *d_moer = nullptr, *d_dgrid = nullptr, *d_sin = nullptr,
         *d_cos = nullptr, *d_catcum = nullptr, *d_pthr = nullptr, *d_dtab = nullptr, *d_portc = nullptr, *d_treec = nullptr;
  int* d_order = nullptr;
  int8_t* d_wk = nullptr;
  int* d_pfull = nullptr;
  Profile* d_prof = nullptr;
  uint32_t* d_err = nullptr;
  unsigned long long* d_tile_ctr = nullptr;
  double thr32 = 0.0;
  vy_state st{};
  vy_outputs out{};
  bool bound = false;
  int64_t launches = 0;
  int smem_per_sm = 0, num_sms = 0;
  int last_mode = -1;  // Spec<M> of the last vy_step launch (diagnostics)
  int tiles_per_warp = 1;  // persistent k_step grid: at most ceil(tiles / (warps per CTA * this)) CTAs
  int wide = -1;           // rollout kernel: 1 warp-per-env (k_rollout_wide), 0 tiles, -1 by batch size
};

namespace {

// per-warp tile layout (see TileLayout); rollouts get a separate obs area
TileLayout tile_layout(const vy_tables& t, bool rollout, bool acts, bool stream = false) {
  TileLayout L{};
  const int n = t.n_ports;
  if (stream) {
    // streamed tile (Spec<4>): i_drawn slots, meta, actions, the obs chunk ring
    L.ps = 256;
    L.ports = 0;
    int off = n * 256;
    L.dtrem = 0;  // dwell times are read from HBM in the port loop
    L.meta = off;
    off += ((n * 32) + 15) & ~15;
    L.acts = off;
    if (acts) off += ((32 * (n + 1)) + 15) & ~15;
    L.obs = (off + 15) & ~15;
    off = L.obs + (kRingBufs == 1 ? kChunkBuf : std::max(2 * kChunkBuf, (9 + t.horizon) * kChunkCol * 4));
    L.bar = (off + 15) & ~15;
    off = L.bar + 16;
    L.bytes = (off + 127) & ~127;
    return L;
  }
  L.ps = 768;
  // the 24n-byte pad lets in-place obs staging (k_step) run ahead of the slots; rollouts stage elsewhere
  L.ports = rollout && kRingBufs == 1 ? 0 : (24 * n + 15) & ~15;
  int off = L.ports + n * 768;
  L.dtrem = off;
  off += n * 64;
  L.meta = off;
  off += ((n * 32) + 15) & ~15;
  L.acts = off;
  if (acts) off += ((32 * (n + 1)) + 15) & ~15;
  const int staging = 132 * t.obs_len;
  L.obs = 0;
  if (rollout) {
    // f32 obs leave through the per-port chunk ring (ObsSink::chunk): two
    // 6-column buffers, also holding the 9 + horizon tail columns
    const int ring = kRingBufs == 1 ? kChunkBuf : std::max(2 * kChunkBuf, (9 + t.horizon) * kChunkCol * 4);
    L.obs = (off + 15) & ~15;
    off = L.obs + ring;
  } else if (off < staging) {
    off = staging;  // in-place staging may run past the state into the dwell/meta/action area
  }
  L.bar = (off + 15) & ~15;
  off = L.bar + 16;
  L.bytes = rollout && kRingBufs == 1 ? (off + 15) & ~15 : (off + 127) & ~127;
  return L;
}

double rcp(double d) { return 1.0 / d; }

// L2 prefetch distance of the streamed step (Params::pf_dist), in tiles: a
// fraction (percent; VY_PF overrides) of the resident warps, i.e. of the tiles
// in flight at once
int g_pf_percent = -1;
int64_t pf_dist(unsigned grid, int warps) {
  if (g_pf_percent < 0) {
    const char* v = std::getenv("VY_PF");
    g_pf_percent = v ? std::atoi(v) : 12;  // 5-25 measured equal, 50+ slower (profiles/r2_c4_prefetch_ab.txt)
  }
  return (int64_t)grid * warps * g_pf_percent / 100;
}

void fill(vy_handle* h, Params& P, bool rollout, bool acts, bool stream = false) {
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
  P.b_rcp_volt = rcp(t.b_volt);
  P.b_rcp_cap = rcp(t.b_cap);
  P.b_rcp_omt = rcp(P.b_omt);
  P.b_rcp_eta_c = rcp(t.b_eta_c);
  P.b_rcp_idenom = rcp(t.b_idenom);
  P.rcp_1000 = rcp(1000.0);
  P.rcp_ep = rcp((double)t.episode_steps);
  P.rcp_365 = rcp(365.0);
  P.battery_node_mask = 0;
  if (t.battery_enabled && t.n_nodes <= kFastNodes)
    for (int m = 0; m < t.n_nodes; ++m)
      if (h->node_lo[m] <= t.n_ports && t.n_ports < h->node_hi[m]) P.battery_node_mask |= 1 << m;
  for (int m = 0; m < t.n_nodes && m < kFastNodes; ++m) {
    P.node_cap[m] = h->node_cap[m];
    P.node_eta[m] = h->node_eta[m];
    P.node_rcp_eta[m] = rcp(h->node_eta[m]);
  }
  P.order = h->d_order;
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
  P.portc = h->d_portc;
  P.treec = h->d_treec;
  P.st = h->st;
  P.out = h->out;
  P.err = h->d_err;
  P.tile_ctr = h->d_tile_ctr;
  P.act_tile = acts;
  P.n_profiles = (int)h->profiles.size();
  P.L = tile_layout(t, rollout, acts, stream);
}

// Warps per CTA: fill the SM's shared memory with as many tiles as possible
// (<= 8 warps per CTA), one CTA per SM if a single tile set is that large.
struct Geometry {
  int warps, smem;
  unsigned grid;
};

// Warps per CTA: fill the SM's shared memory with as many warp tiles as
// possible (several CTAs per SM when they fit, else one large CTA).
template <typename K>
int geometry(vy_handle* h, K kernel, const TileLayout& L, int n_profiles, Geometry& g) {
  const int per_sm = h->smem_per_sm;
  const int tb = tables_bytes(n_profiles, h->t.k, h->t.n_ports, h->t.n_nodes);
  int best_w = 1, best_total = 0;
  for (int w = 1; w <= 8; ++w) {  // __launch_bounds__(256)
    const int bytes = tb + w * L.bytes;
    if (bytes + 1024 > per_sm) break;
    const int blocks = per_sm / (bytes + 1024);
    const int total = blocks * w;
    if (blocks >= 1 && total >= best_total) {  // ties: prefer larger CTAs (fewer table copies)
      best_total = total;
      best_w = w;
    }
  }
  if (const char* ov = std::getenv("VY_WARPS_PER_CTA")) {  // tuning override
    const int w = std::atoi(ov);
    if (w >= 1 && w <= 8 && tb + w * L.bytes + 1024 <= per_sm) best_w = w;
  }
  g.warps = best_w;
  g.smem = tb + best_w * L.bytes;
  if (g.smem + 1024 > per_sm) return fail(VY_ERR_UNSUPPORTED, "station too large for one shared-memory tile");
  if (g.smem > 48 * 1024)
    VY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem));
  const int64_t tiles = (h->B + 31) / 32;
  g.grid = (unsigned)((tiles + best_w - 1) / best_w);
  return VY_OK;
}

// Which Spec<M> (vy_device.cuh) a call runs: 1 or 2 (lean, small or large
// tree) for lean outputs without any of the optional model features, an
// identity-ordered station and a shuffle-sized grid; 3 the same with a
// battery; 0 (generic) otherwise.
int step_mode(const vy_handle* h, uint32_t flags, bool staged_actions) {
  const vy_tables& t = h->t;
  const bool lean = (flags & ~VY_F_AUTO_RESET) == 0 && staged_actions && !t.has_moer && !t.has_dgrid &&
                    t.horizon == 0 && h->order_identity && 2 * t.k < 32;
  if (!lean) return 0;
  // battery stations: large ones (config C4, 64 ports: a 62 KB resident tile,
  // 3 warps per SM) stream their tile (4), small ones keep it resident (3)
  if (t.battery_enabled) return t.n_ports > 16 ? 4 : 3;
  return t.n_nodes <= kFastNodes ? 1 : 2;
}

Profile make_profile(double cap, double r_ac, double r_dc, double tau) {
  const double omt = 1.0 - tau;
  return Profile{cap, r_ac, r_dc, tau, omt, 1.0 / cap, 1.0 / omt, 0.0, 0.0};
}

int upload_profiles(vy_handle* h) {
  std::vector<Profile> all(kMaxProfiles, Profile{1.0, 0.0, 0.0, 0.5, 0.5, 1.0, 2.0, 0.0, 0.0});
  for (size_t i = 0; i < h->profiles.size(); ++i) all[i] = h->profiles[i];
  VY_CUDA(cudaMemcpy(h->d_prof, all.data(), sizeof(Profile) * kMaxProfiles, cudaMemcpyHostToDevice));
  return VY_OK;
}

}  // namespace

extern "C" {

int vy_abi_version(void) { return VY_ABI_VERSION; }
const char* vy_last_error(void) { return g_err.c_str(); }

int vy_create(const vy_tables* t, int64_t batch, int device, vy_handle** out) {
  if (!t || !out) return fail(VY_ERR_ARG, "null argument");
  if (batch < 1) return fail(VY_ERR_ARG, "batch_size must be >= 1");
  const int n = t->n_ports;
  if (n < 1 || n > 64) return fail(VY_ERR_UNSUPPORTED, "n_ports must be in [1, 64]");
  if (t->n_cat < 1 || t->n_cat > kMaxProfiles) return fail(VY_ERR_UNSUPPORTED, "catalogue must hold 1..64 cars");
  if ((int64_t)t->episode_steps + t->stay_hi > 32000 || t->stay_hi > 32000)
    return fail(VY_ERR_UNSUPPORTED, "stay / episode lengths exceed the int16 dwell-time state");
  if (t->n_days < 1 || t->lam_len < 1 || t->steps_per_day < 1) return fail(VY_ERR_ARG, "empty series");
  if (t->dt_min < 1 || t->dt_min > 1440 || t->episode_steps < 1)
    return fail(VY_ERR_ARG, "dt_min must be in [1, 1440] and episode_steps >= 1");
  vy_handle* h = new vy_handle();
  h->device = device;
  h->B = batch;
  h->t = *t;
  if (t->n_nodes > kMaxNodes) {
    delete h;
    return fail(VY_ERR_UNSUPPORTED, "too many tree nodes for the compiled capacity");
  }
  h->volt.assign(t->volt, t->volt + n);
  h->imax_c.assign(t->imax_c, t->imax_c + n);
  h->imax_d.assign(t->imax_d, t->imax_d + n);
  h->eta_c.assign(t->eta_c, t->eta_c + n);
  h->eta_d.assign(t->eta_d, t->eta_d + n);
  h->i_denom.assign(t->i_denom, t->i_denom + n);
  h->kind.assign(t->kind, t->kind + n);
  h->order.assign(t->order, t->order + n);
  for (int i = 0; i < n; ++i) h->order_identity &= h->order[i] == i;
  // tree: contiguous leaf ranges (topology.py:178-196)
  for (int m = 0; m < t->n_nodes; ++m) {
    const int a0 = t->node_ptr[m], a1 = t->node_ptr[m + 1];
    int lo = 0, hi = 0;
    if (a1 > a0) {
      lo = t->node_leaf[a0];
      hi = lo + (a1 - a0);
      for (int a = a0; a < a1; ++a)
        if (t->node_leaf[a] != lo + (a - a0)) {
          delete h;
          return fail(VY_ERR_UNSUPPORTED, "tree node leaves are not one ascending run");
        }
    }
    if (hi > t->n_slots) {
      delete h;
      return fail(VY_ERR_ARG, "tree leaf index out of range");
    }
    h->node_lo.push_back(lo);
    h->node_hi.push_back(hi);
    h->node_cap.push_back(t->node_cap[m]);
    h->node_eta.push_back(t->node_eta[m]);
    h->node_order.push_back(t->node_order[m]);
  }
  for (int c = 0; c < t->n_cat; ++c) {
    h->profiles.push_back(make_profile(t->cat_cap[c], t->cat_rac[c], t->cat_rdc[c], t->cat_tau[c]));
    h->profiles.back().cum = t->cat_cum[c];
  }
  // Poisson: per (weekday flag, step-of-profile) the number of full 32-chunks and the
  // threshold of the last chunk, reproducing rng.py:94-115 / _kernel.pyx:55-73 on the host.
  const int L = t->lam_len;
  std::vector<double> pthr(2 * L, 0.0);
  std::vector<int> pfull(2 * L, -1);
  for (int w = 0; w < 2; ++w)
    for (int j = 0; j < L; ++j) {
      double lam = t->lam[j] * (w == 0 ? t->wk_scale : t->we_scale);
      if (lam <= 0.0) continue;
      int full = 0;
      while (lam > 32.0) {
        lam -= 32.0;
        ++full;
      }
      pfull[w * L + j] = full;
      pthr[w * L + j] = std::exp(-lam);
    }
  h->thr32 = std::exp(-32.0);
  const int nd = 2 * t->k + 1;
  std::vector<double> dtab(nd);
  for (int a = 0; a < nd; ++a) dtab[a] = (double)(a - t->k) / (double)t->k;
  int rc = cudaSetDevice(device) == cudaSuccess ? VY_OK : fail(VY_ERR_CUDA, "cudaSetDevice failed");
  if (!rc && cudaDeviceGetAttribute(&h->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device) != cudaSuccess)
    rc = fail(VY_ERR_CUDA, "device query failed");
  if (!rc && cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    rc = fail(VY_ERR_CUDA, "device query failed");
  const size_t nh = (size_t)t->n_days * 24;
  if (!rc) rc = upload(&h->d_buy, t->buy, nh);
  if (!rc) rc = upload(&h->d_sellg, t->sellg, nh);
  if (!rc) rc = upload(&h->d_moer, t->moer, t->has_moer ? nh : 1);
  if (!rc) rc = upload(&h->d_dgrid, t->dgrid, t->has_dgrid ? nh : 1);
  if (!rc) rc = upload(&h->d_sin, t->sin_t, (size_t)t->steps_per_day);
  if (!rc) rc = upload(&h->d_cos, t->cos_t, (size_t)t->steps_per_day);
  if (!rc) rc = upload(&h->d_catcum, t->cat_cum, (size_t)t->n_cat);
  if (!rc) rc = upload(&h->d_wk, t->weekday, (size_t)t->n_days);
  if (!rc) rc = upload(&h->d_pthr, pthr.data(), pthr.size());
  if (!rc) rc = upload(&h->d_pfull, pfull.data(), pfull.size());
  if (!rc) rc = upload(&h->d_dtab, dtab.data(), dtab.size());
  {
    // per-port constant records (PortC, vy_tile.cuh)
    std::vector<double> pcv((size_t)n * kPortWords);
    for (int i = 0; i < n; ++i) {
      double* r = pcv.data() + (size_t)i * kPortWords;
      uint32_t mask = 0;
      for (int m = 0; m < t->n_nodes && m < kFastNodes; ++m)
        if (h->node_lo[m] <= i && i < h->node_hi[m]) mask |= 1u << m;
      const double dtv = t->dt_h * t->volt[i];
      r[0] = t->imax_c[i], r[1] = t->imax_d[i], r[2] = t->volt[i], r[3] = rcp(t->volt[i]);
      r[4] = t->kind[i] ? 1.0 : 0.0, r[5] = t->n_nodes <= kFastNodes ? (double)mask : 0.0;
      r[6] = dtv, r[7] = t->eta_d[i], r[8] = t->eta_c[i], r[9] = rcp(t->eta_c[i]);
      r[10] = t->i_denom[i], r[11] = rcp(t->i_denom[i]);
    }
    if (!rc) rc = upload(&h->d_portc, pcv.data(), pcv.size());
    // tree records in the deepest-first rescale order (TreeC, vy_tile.cuh)
    std::vector<double> tcv((size_t)(t->n_nodes > 0 ? t->n_nodes : 1) * 4, 0.0);
    for (int q = 0; q < t->n_nodes; ++q) {
      const int m = h->node_order[q];
      double* r = tcv.data() + (size_t)q * 4;
      r[0] = h->node_cap[m], r[1] = h->node_eta[m], r[2] = rcp(h->node_eta[m]);
      const int32_t lohi[2] = {h->node_lo[m], h->node_hi[m]};
      std::memcpy(&r[3], lohi, 8);
    }
    if (!rc) rc = upload(&h->d_treec, tcv.data(), tcv.size());
  }
  if (!rc) rc = upload(&h->d_order, h->order.data(), h->order.size());
  if (!rc) rc = upload<Profile>(&h->d_prof, nullptr, kMaxProfiles);
  if (!rc) rc = upload<uint32_t>(&h->d_err, nullptr, 1);
  if (!rc && cudaMemset(h->d_err, 0, 4) != cudaSuccess) rc = fail(VY_ERR_CUDA, "memset");
  if (!rc) rc = upload<unsigned long long>(&h->d_tile_ctr, nullptr, 2);
  if (!rc && cudaMemset(h->d_tile_ctr, 0, 16) != cudaSuccess) rc = fail(VY_ERR_CUDA, "memset");
  if (!rc) rc = upload_profiles(h);
  if (rc) {
    vy_destroy(h);
    return rc;
  }
  *out = h;
  return VY_OK;
}

int vy_destroy(vy_handle* h) {
  if (!h) return VY_OK;
  void* ptrs[] = {h->d_buy, h->d_sellg, h->d_moer, h->d_dgrid, h->d_sin, h->d_cos, h->d_catcum,
                  h->d_pthr, h->d_dtab, h->d_portc, h->d_treec, h->d_wk, h->d_pfull, h->d_prof, h->d_err, h->d_tile_ctr,
                  h->d_order};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete h;
  return VY_OK;
}

int vy_add_profile(vy_handle* h, double cap, double r_ac, double r_dc, double tau) {
  if (!h || (int)h->profiles.size() >= kMaxProfiles) {
    fail(VY_ERR_ARG, "profile table full");
    return -1;
  }
  if (!(cap > 0.0) || !(tau > 0.0 && tau < 1.0)) {
    fail(VY_ERR_ARG, "profile needs cap > 0 and 0 < tau < 1");
    return -1;
  }
  for (size_t i = 0; i < h->profiles.size(); ++i) {
    const Profile& p = h->profiles[i];
    if (p.cap == cap && p.r_ac == r_ac && p.r_dc == r_dc && p.tau == tau) return (int)i;
  }
  h->profiles.push_back(make_profile(cap, r_ac, r_dc, tau));
  if (upload_profiles(h)) return -1;
  return (int)h->profiles.size() - 1;
}

int vy_get_profile(vy_handle* h, int p, double out4[4]) {
  if (!h || p < 0 || p >= (int)h->profiles.size()) return fail(VY_ERR_ARG, "bad profile id");
  out4[0] = h->profiles[p].cap;
  out4[1] = h->profiles[p].r_ac;
  out4[2] = h->profiles[p].r_dc;
  out4[3] = h->profiles[p].tau;
  return VY_OK;
}

int vy_bind(vy_handle* h, const vy_state* s, const vy_outputs* o) {
  if (!h || !s || !o) return fail(VY_ERR_ARG, "null argument");
  if (s->ld < ((h->B + 31) / 32) * 32 || s->ld % 32)
    return fail(VY_ERR_ARG, "state leading dimension must be a multiple of 32 covering the batch");
  if (!s->port_i || !s->port_soc || !s->port_de || !s->port_dtrem || !s->port_meta || !s->step || !s->day ||
      !s->episode || !s->env_seed || !s->akey || !s->b_i || !s->b_soc || !s->ep_profit || !s->ep_reward ||
      !s->ep_missing || !s->ep_energy || !s->ep_overtime || !s->ep_declined || !s->ep_departures)
    return fail(VY_ERR_ARG, "state buffer missing");
  if (!o->obs || !o->reward || !o->done || !o->ep_stats || !o->term_overtime)
    return fail(VY_ERR_ARG, "output buffer missing");
  h->st = *s;
  h->out = *o;
  h->bound = true;
  return VY_OK;
}

static bool infos_bound(const vy_outputs& o) {
  return o.breakdown && o.flows && o.declined && o.arrivals_m && o.dep_n && o.dep_port && o.dep_overtime &&
         o.dep_early && o.dep_pref && o.dep_missing && o.dep_cap && o.dep_soc && o.i_att && o.i_used &&
         o.delivered && o.b_delivered;
}

int vy_reset(vy_handle* h, const uint8_t* mask, int32_t episode_mode, const int32_t* inj_day, uint32_t flags,
             void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  Params P;
  fill(h, P, false, false);
  P.flags = flags;
  Geometry g;
  if (int rc = geometry(h, k_reset, P.L, P.n_profiles, g)) return rc;
  k_reset<<<g.grid, g.warps * 32, g.smem, (cudaStream_t)stream>>>(P, mask, episode_mode, inj_day, nullptr);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_reset_episodes(vy_handle* h, const uint8_t* mask, const int32_t* episodes, uint32_t flags, void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  if (!episodes) return fail(VY_ERR_ARG, "null episodes");
  Params P;
  fill(h, P, false, false);
  P.flags = flags;
  Geometry g;
  if (int rc = geometry(h, k_reset, P.L, P.n_profiles, g)) return rc;
  k_reset<<<g.grid, g.warps * 32, g.smem, (cudaStream_t)stream>>>(P, mask, 0, nullptr, episodes);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_seed_envs(vy_handle* h, int64_t master_seed, int64_t index0, void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  const unsigned grid = (unsigned)((h->B + 255) / 256);
  k_seed_envs<<<grid, 256, 0, (cudaStream_t)stream>>>((uint64_t)master_seed, index0, h->B, h->st.env_seed);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_step(vy_handle* h, const void* actions, int32_t dtype, int64_t row_stride, int64_t col_stride,
            uint32_t flags, const vy_draws* inj, void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  if (!actions) return fail(VY_ERR_ARG, "null actions");
  if (dtype != VY_ACT_U8 && dtype != VY_ACT_I32 && dtype != VY_ACT_I64) return fail(VY_ERR_ARG, "bad action dtype");
  if ((flags & VY_F_INFOS) && !infos_bound(h->out)) return fail(VY_ERR_ARG, "info buffers not bound");
  if ((flags & VY_F_INJECT) && (!inj || !inj->off || !inj->profile || !inj->stay || !inj->soc0 || !inj->frac ||
                                !inj->pref))
    return fail(VY_ERR_ARG, "injected draws missing");
  // stage the action block per tile when it is the canonical uint8 [B][n+1] row-major
  // layout: 16-byte aligned per tile and over-reading whole chunks stays in bounds
  const int na = h->t.n_ports + 1;
  const bool acts = dtype == VY_ACT_U8 && col_stride == 1 && row_stride == na &&
                    (reinterpret_cast<uintptr_t>(actions) % 16) == 0 && (32 * na) % 16 == 0 &&
                    (h->B % 32) == 0;
  const int mode = step_mode(h, flags, acts);
  // small batches: the one-warp-per-env kernel for a single step (auto-reset on, staged uint8 rows),
  // when the handle asks for it (vy_set_wide(h, 1); the PPO trainer does at its batch sizes)
  if ((mode == 1 || mode == 2) && flags == VY_F_AUTO_RESET && h->t.n_ports <= 32 && h->wide == 1) {
    Params P;
    fill(h, P, true, false);
    P.flags = flags;
    const int smem = tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes) + kWideWarps * kWideScratch * 8;
    auto* kern = mode == 1 ? k_rollout_wide<1> : k_rollout_wide<2>;
    if (smem > 48 * 1024) VY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)((h->B + kWideWarps - 1) / kWideWarps);
    kern<<<grid, 32 * kWideWarps, smem, (cudaStream_t)stream>>>(P, 1, 0, 0, 0, 0, 0,
                                                                  static_cast<const uint8_t*>(actions));
    VY_CUDA(cudaGetLastError());
    ++h->launches;
    h->last_mode = 10 + mode;
    return VY_OK;
  }
  Params P;
  fill(h, P, false, acts, mode == 4);
  P.flags = flags;
  P.actions = actions;
  P.act_dtype = dtype;
  P.act_row = row_stride;
  P.act_col = col_stride;
  if (inj) P.inj = *inj;
  Geometry g;
  h->last_mode = mode;
  auto* kern = mode == 1 ? k_step<1> : mode == 2 ? k_step<2> : mode == 3 ? k_step<3> : mode == 4 ? k_step<4> : k_step<0>;
  if (int rc = geometry(h, kern, P.L, P.n_profiles, g)) return rc;
  // persistent grid: every resident CTA slot, never more CTAs than tiles need
  const unsigned resident = (unsigned)h->num_sms * (unsigned)(h->smem_per_sm / (g.smem + 1024));
  unsigned grid = g.grid < resident ? g.grid : resident;
  if (h->tiles_per_warp > 1) {  // fewer, longer-lived warps (batches sharing the GPU)
    const unsigned k = (unsigned)h->tiles_per_warp, want = (g.grid + k - 1) / k;
    grid = want < grid ? want : grid;
  }
  if (mode == 4) P.pf_dist = pf_dist(grid, g.warps);
  kern<<<grid, g.warps * 32, g.smem, (cudaStream_t)stream>>>(P);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_step_random(vy_handle* h, uint64_t seed, int64_t index0, int64_t call, int64_t* call_counter,
                   uint8_t* actions_out, uint32_t flags, void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  if ((flags & VY_F_INFOS) && !infos_bound(h->out)) return fail(VY_ERR_ARG, "info buffers not bound");
  if (flags & VY_F_INJECT) return fail(VY_ERR_UNSUPPORTED, "vy_step_random draws its own arrivals (no VY_F_INJECT)");
  if (2 * h->t.k + 1 > 256) return fail(VY_ERR_UNSUPPORTED, "RandomPolicy actions need 2k+1 <= 256");
  const int mode = step_mode(h, flags, true);
  Params P;
  fill(h, P, false, true, mode == 4);  // the generated rows live in the tile's staged-action area
  P.flags = flags;
  P.actions = nullptr;
  P.act_dtype = VY_ACT_U8;
  P.policy = 1;
  P.pol_seed = seed;
  P.pol_index0 = index0;
  P.pol_call = call;
  P.pol_counter = call_counter;
  P.pol_out = actions_out;
  Geometry g;
  h->last_mode = mode;
  auto* kern = mode == 1 ? k_step<1> : mode == 2 ? k_step<2> : mode == 3 ? k_step<3> : mode == 4 ? k_step<4> : k_step<0>;
  if (int rc = geometry(h, kern, P.L, P.n_profiles, g)) return rc;
  const unsigned resident = (unsigned)h->num_sms * (unsigned)(h->smem_per_sm / (g.smem + 1024));
  unsigned grid = g.grid < resident ? g.grid : resident;
  if (h->tiles_per_warp > 1) {
    const unsigned k = (unsigned)h->tiles_per_warp, want = (g.grid + k - 1) / k;
    grid = want < grid ? want : grid;
  }
  if (mode == 4) P.pf_dist = pf_dist(grid, g.warps);
  kern<<<grid, g.warps * 32, g.smem, (cudaStream_t)stream>>>(P);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_random_actions(vy_handle* h, uint64_t seed, int64_t index0, int64_t call, uint8_t* out, void* stream) {
  if (!h || !out) return fail(VY_ERR_ARG, "null argument");
  const int ns = h->t.n_ports + 1, hi = 2 * h->t.k + 1;
  if (hi > 256) return fail(VY_ERR_UNSUPPORTED, "uint8 actions need 2k+1 <= 256");
  const unsigned grid = (unsigned)((h->B + 255) / 256);
  k_random_actions<<<grid, 256, 8 * 32 * ns, (cudaStream_t)stream>>>(seed, index0, call, h->B, ns, hi, out,
                                                                     nullptr);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_random_actions_dev(vy_handle* h, uint64_t seed, int64_t index0, int64_t* call_counter, uint8_t* out,
                          void* stream) {
  if (!h || !out || !call_counter) return fail(VY_ERR_ARG, "null argument");
  const int ns = h->t.n_ports + 1, hi = 2 * h->t.k + 1;
  if (hi > 256) return fail(VY_ERR_UNSUPPORTED, "uint8 actions need 2k+1 <= 256");
  const unsigned grid = (unsigned)((h->B + 255) / 256);
  k_random_actions<<<grid, 256, 8 * 32 * ns, (cudaStream_t)stream>>>(seed, index0, 0, h->B, ns, hi, out,
                                                                     call_counter);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_rollout(vy_handle* h, int32_t T, uint64_t policy_seed, int64_t index0, int64_t call0, void* obs,
               int64_t obs_step_stride, void* reward, uint8_t* done, int64_t rew_step_stride, uint32_t flags,
               void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  if (T < 1 || !obs || !reward || !done) return fail(VY_ERR_ARG, "bad rollout arguments");
  if (flags & (VY_F_INFOS | VY_F_INJECT)) return fail(VY_ERR_UNSUPPORTED, "rollout supports lean outputs only");
  if (2 * h->t.k + 1 > 256) return fail(VY_ERR_UNSUPPORTED, "rollout needs 2k+1 <= 256");
  Params P;
  fill(h, P, true, false);
  P.flags = flags;
  P.out.obs = obs;
  P.out.reward = reward;
  P.out.done = done;
  Geometry g;
  int mode = step_mode(h, flags, true);
  // small batches: one warp per env, one lane per port (vy_wide.cuh) — lean
  // stations without a battery, <= 32 ports; by default up to 4096 envs, where
  // the tile kernel is latency-bound (16 envs: 3.2 vs 10 us per step; 4096:
  // 8.3 vs 12.2 us, scripts/probe_c1.py)
  const bool wide_ok = (mode == 1 || mode == 2) && h->t.n_ports <= 32 && !(flags & VY_F_OUT_F64);
  if (wide_ok && (h->wide == 1 || (h->wide < 0 && h->B <= 4096))) {
    Params P;
    fill(h, P, true, false);
    P.flags = flags;
    P.out.obs = obs;
    P.out.reward = reward;
    P.out.done = done;
    const int smem = tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes) + kWideWarps * kWideScratch * 8;
    auto* kern = mode == 1 ? k_rollout_wide<1> : k_rollout_wide<2>;
    if (smem > 48 * 1024) VY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)((h->B + kWideWarps - 1) / kWideWarps);
    kern<<<grid, 32 * kWideWarps, smem, (cudaStream_t)stream>>>(P, T, policy_seed, index0, call0, obs_step_stride,
                                                                  rew_step_stride, nullptr);
    VY_CUDA(cudaGetLastError());
    ++h->launches;
    h->last_mode = 10 + mode;  // diagnostics: 11 / 12 = wide rollout
    return VY_OK;
  }
  if (mode == 4) mode = 3;  // a rollout keeps the whole tile resident for its T steps
  auto* kern = mode == 1 ? k_rollout<1> : mode == 2 ? k_rollout<2> : mode == 3 ? k_rollout<3> : k_rollout<0>;
  if (int rc = geometry(h, kern, P.L, P.n_profiles, g)) return rc;
  kern<<<g.grid, g.warps * 32, g.smem, (cudaStream_t)stream>>>(P, T, policy_seed, index0, call0, obs_step_stride,
                                                              rew_step_stride);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  return VY_OK;
}

int vy_poll_error(vy_handle* h, int clear, void* stream, uint32_t* out) {
  if (!h || !out) return fail(VY_ERR_ARG, "null argument");
  VY_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  VY_CUDA(cudaMemcpy(out, h->d_err, 4, cudaMemcpyDeviceToHost));
  if (clear) VY_CUDA(cudaMemset(h->d_err, 0, 4));
  return VY_OK;
}

int64_t vy_launch_count(vy_handle* h) { return h ? h->launches : -1; }
int32_t vy_last_step_mode(vy_handle* h) { return h ? h->last_mode : -1; }

int vy_ppo_rollout(vy_handle* h, int32_t T, const void* wpack, const float* fpack, int32_t S, int32_t A,
                   uint64_t seed, int64_t* counter, float* obs, uint8_t* actions, float* logp, float* value,
                   float* reward, uint8_t* done, void* stream) {
  if (!h || !h->bound) return fail(VY_ERR_STATE, "handle not bound");
  if (T < 1 || !wpack || !fpack || !counter || !obs || !actions || !logp || !value || !reward || !done)
    return fail(VY_ERR_ARG, "bad PPO rollout arguments");
  if (((reinterpret_cast<uintptr_t>(wpack) | reinterpret_cast<uintptr_t>(fpack)) & 15u) != 0)
    return fail(VY_ERR_ARG, "weight packs must be 16-byte aligned");
  // the env side is the one-warp-per-env step: lean stations without a battery, <= 32 ports
  const int mode = step_mode(h, VY_F_AUTO_RESET, true);
  if (!(mode == 1 || mode == 2) || h->t.n_ports > 32 || S != h->t.n_ports + 1)
    return fail(VY_ERR_UNSUPPORTED, "fused PPO rollout needs a lean station without a battery, <= 32 ports");
  const int OL = h->t.obs_len;
  int32_t geo[4];
  if (vy_policy_geometry(OL, OL, S, A, geo) != VY_OK) return fail(VY_ERR_UNSUPPORTED, "policy geometry");
  if (A != 2 * h->t.k + 1) return fail(VY_ERR_ARG, "actions per slot must be 2k+1");
  const vyp::Geo g = vyp::make_geo(OL, OL, S, A);
  Params P;
  fill(h, P, true, false);
  P.flags = VY_F_AUTO_RESET;
  P.out.reward = reward;
  P.out.done = done;
  const uint32_t pol = ppo_policy_off(ppo_scratch_off(P.n_profiles, P.k, P.n_ports, P.n_nodes));
  const int smem = (int)(pol + g.smem);
  if (smem > 227 * 1024) return fail(VY_ERR_UNSUPPORTED, "fused PPO rollout: shared memory");
  auto* kern = mode == 1 ? k_ppo_rollout<1> : k_ppo_rollout<2>;
  VY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  PpoBufs R{static_cast<const uint8_t*>(wpack), fpack, seed, reinterpret_cast<unsigned long long*>(counter),
            obs, actions, logp, value};
  // envs per CTA: as few as one wave of CTAs allows (fewer env warps per SM
  // step faster; the policy pass costs the same for 1 or 16 rows), at least 2
  // (16 envs: 8.9 us per step at 2-4 per CTA, 10.0 at 16; scripts/gpu_r2_ppo_epc.sh)
  const int64_t per = (h->B + h->num_sms - 1) / h->num_sms;
  int epc = per < 2 ? 2 : (per > kPpoEnvs ? kPpoEnvs : (int)per);
  if (const char* e = getenv("VY_PPO_EPC")) epc = atoi(e) < 1 ? 1 : (atoi(e) > kPpoEnvs ? kPpoEnvs : atoi(e));
  const unsigned grid = (unsigned)((h->B + epc - 1) / epc);
  kern<<<grid, kPpoThreads, smem, (cudaStream_t)stream>>>(P, T, epc, g, R);
  VY_CUDA(cudaGetLastError());
  ++h->launches;
  h->last_mode = 20 + mode;  // diagnostics: 21 / 22 = fused PPO rollout
  return VY_OK;
}

#ifdef VY_PPO_PROF
int vy_ppo_prof_read(unsigned long long* out) {
  VY_CUDA(cudaMemcpyFromSymbol(out, g_ppo_prof, sizeof(g_ppo_prof)));
  return VY_OK;
}
int vy_env_stamps_read(unsigned long long* out) {
  VY_CUDA(cudaMemcpyFromSymbol(out, g_env_stamp, sizeof(g_env_stamp)));
  return VY_OK;
}
#endif

int vy_set_wide(vy_handle* h, int32_t mode) {
  if (!h || mode < -1 || mode > 1) return fail(VY_ERR_ARG, "wide mode must be -1 (auto), 0 or 1");
  h->wide = mode;
  return VY_OK;
}

int vy_set_tiles_per_warp(vy_handle* h, int32_t k) {
  if (!h || k < 1) return fail(VY_ERR_ARG, "tiles per warp must be >= 1");
  h->tiles_per_warp = k;
  return VY_OK;
}

int vy_selftest_div(const double* divisors, int32_t nd, int64_t samples_per_divisor, uint64_t seed,
                    int64_t* mismatches) {
  if (!divisors || nd < 1 || samples_per_divisor < 1 || !mismatches) return fail(VY_ERR_ARG, "bad arguments");
  std::vector<double> y(nd);
  for (int i = 0; i < nd; ++i) {
    if (!(divisors[i] > 0.0)) return fail(VY_ERR_ARG, "divisors must be positive");
    y[i] = 1.0 / divisors[i];
  }
  double *dd = nullptr, *dy = nullptr;
  unsigned long long* dbad = nullptr;
  int rc = upload(&dd, divisors, (size_t)nd);
  if (!rc) rc = upload(&dy, y.data(), (size_t)nd);
  if (!rc) rc = upload<unsigned long long>(&dbad, nullptr, 1);
  if (!rc && cudaMemset(dbad, 0, 8) != cudaSuccess) rc = fail(VY_ERR_CUDA, "memset");
  if (!rc) {
    k_selftest_div<<<148 * 8, 256>>>(dd, dy, nd, samples_per_divisor, seed, dbad);
    unsigned long long bad = 0;
    if (cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost) != cudaSuccess) rc = fail(VY_ERR_CUDA, "selftest failed");
    *mismatches = (int64_t)bad;
  }
  cudaFree(dd);
  cudaFree(dy);
  cudaFree(dbad);
  return rc;
}

}  // extern "C"

// ---- heterogeneous batch in one launch (k_step_multi) ---------------------

struct vy_multi {
  std::vector<vy_handle*> hs;
  int mode = 1;
  vy::MultiArgs A{};
  unsigned long long* d_ctr = nullptr;
  int smem = 0, warps = 1;
  unsigned grid = 0;
  int64_t launches = 0;
};

namespace {
// c_groups slots in use (constant memory is per module: live multi handles share it)
std::mutex g_slot_mu;
std::vector<bool> g_slot_used(kConstGroups, false);
int alloc_slots(int n) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  for (int s0 = 0; s0 + n <= kConstGroups; ++s0) {
    bool ok = true;
    for (int j = 0; j < n && ok; ++j) ok = !g_slot_used[(size_t)(s0 + j)];
    if (ok) {
      for (int j = 0; j < n; ++j) g_slot_used[(size_t)(s0 + j)] = true;
      return s0;
    }
  }
  return -1;
}
void free_slots(int s0, int n) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  for (int j = 0; j < n; ++j) g_slot_used[(size_t)(s0 + j)] = false;
}
// the bytes of a group's car-profile table / station tables (action grid,
// per-port constants, capacity tree): groups with equal bytes share one
// staged copy per CTA
int profile_bytes_of(const Params& P, std::vector<unsigned char>& out) {
  const size_t np = (size_t)P.n_profiles * sizeof(Profile);
  out.assign(4 + np, 0);
  std::memcpy(out.data(), &P.n_profiles, 4);
  VY_CUDA(cudaMemcpy(out.data() + 4, P.profiles, np, cudaMemcpyDeviceToHost));
  return VY_OK;
}
int station_bytes_of(const Params& P, std::vector<unsigned char>& out) {
  const size_t nd = (size_t)(2 * P.k + 1) * 8, npc = (size_t)P.n_ports * 8 * kPortWords, nt = (size_t)P.n_nodes * 32;
  out.assign(12 + nd + npc + nt, 0);
  const int32_t dims[3] = {P.k, P.n_ports, P.n_nodes};
  std::memcpy(out.data(), dims, 12);
  unsigned char* o = out.data() + 12;
  VY_CUDA(cudaMemcpy(o, P.delta_tab, nd, cudaMemcpyDeviceToHost));
  VY_CUDA(cudaMemcpy(o + nd, P.portc, npc, cudaMemcpyDeviceToHost));
  VY_CUDA(cudaMemcpy(o + nd + npc, P.treec, nt, cudaMemcpyDeviceToHost));
  return VY_OK;
}
// index of `key` in `sets` (appended if new; -1 when full)
int intern_set(std::vector<std::vector<unsigned char>>& sets, const std::vector<unsigned char>& key) {
  for (size_t s = 0; s < sets.size(); ++s)
    if (sets[s] == key) return (int)s;
  if ((int)sets.size() == kMaxSets) return -1;
  sets.push_back(key);
  return (int)sets.size() - 1;
}
}  // namespace

extern "C" {

int vy_multi_create(vy_handle* const* hs, int32_t n, const uint64_t* policy_seeds, const int64_t* index0,
                    vy_multi** out) {
  if (!hs || !out || !policy_seeds || !index0 || n < 1) return fail(VY_ERR_ARG, "bad arguments");
  if (n > kConstGroups) return fail(VY_ERR_UNSUPPORTED, "at most 48 groups per multi batch");
  auto m = std::make_unique<vy_multi>();
  std::vector<Params> ps((size_t)n);
  std::vector<std::vector<unsigned char>> psets, ssets;
  int mode = 1;
  int device = -1;
  bool battery = false, generic = false, big_tree = false;
  int64_t tiles = 0;
  int tile_bytes = 0;
  for (int g = 0; g < n; ++g) {
    vy_handle* h = hs[g];
    if (!h || !h->bound) return fail(VY_ERR_STATE, "every group handle must be bound");
    if (device < 0) device = h->device;
    if (h->device != device) return fail(VY_ERR_ARG, "groups on different devices");
    if (2 * h->t.k + 1 > 256) return fail(VY_ERR_UNSUPPORTED, "RandomPolicy actions need 2k+1 <= 256");
    const int md = step_mode(h, VY_F_AUTO_RESET, true);
    generic |= md == 0;
    battery |= md == 3 || md == 4;  // the multi launch keeps tiles resident (Spec<3>)
    big_tree |= md == 2;
    Params& P = ps[(size_t)g];
    fill(h, P, false, true);
    P.flags = VY_F_AUTO_RESET;
    P.actions = nullptr;
    P.act_dtype = VY_ACT_U8;
    P.policy = 1;
    P.pol_seed = policy_seeds[g];
    P.pol_index0 = index0[g];
    P.pol_call = 0;
    P.pol_counter = nullptr;
    P.pol_out = nullptr;
    m->A.tile0[g] = tiles;
    tiles += (h->B + 31) / 32;
    tile_bytes = std::max(tile_bytes, P.L.bytes);
    std::vector<unsigned char> key;
    const size_t np0 = psets.size(), ns0 = ssets.size();
    if (int rc = profile_bytes_of(P, key)) return rc;
    const int ps_ = intern_set(psets, key);
    if (int rc = station_bytes_of(P, key)) return rc;
    const int ss_ = intern_set(ssets, key);
    if (ps_ < 0 || ss_ < 0) return fail(VY_ERR_UNSUPPORTED, "at most 8 distinct car-profile / station table sets");
    if (psets.size() > np0) m->A.pset_group[ps_] = g;  // a new set: this group's tables define it
    if (ssets.size() > ns0) m->A.sset_group[ss_] = g;
    m->A.group_pset[g] = (int8_t)ps_;
    m->A.group_sset[g] = (int8_t)ss_;
    m->hs.push_back(h);
  }
  // one Spec<M> for all groups: M = 2 runs any tree (node sums from the tile),
  // M = 3 adds the battery, M = 0 everything else
  mode = generic ? 0 : battery ? 3 : big_tree ? 2 : 1;
  if (battery && big_tree) mode = 3;
  m->mode = mode;
  m->A.n_groups = n;
  m->A.n_psets = (int)psets.size();
  m->A.n_ssets = (int)ssets.size();
  m->A.tile0[n] = tiles;
  int off = 0;
  for (int s = 0; s < m->A.n_psets; ++s) {
    m->A.pset_off[s] = off;
    off += pset_bytes(ps[(size_t)m->A.pset_group[s]].n_profiles);
  }
  for (int s = 0; s < m->A.n_ssets; ++s) {
    const Params& P = ps[(size_t)m->A.sset_group[s]];
    m->A.sset_off[s] = off;
    off += sset_bytes(P.k, P.n_ports, P.n_nodes);
  }
  off = (off + 127) & ~127;
  m->A.tiles_off = off;
  m->A.tile_bytes = (tile_bytes + 16 + 127) & ~127;  // + the warp's mbarrier at the end
  VY_CUDA(cudaSetDevice(device));
  const int slot0 = alloc_slots(n);
  if (slot0 < 0) return fail(VY_ERR_UNSUPPORTED, "constant-memory group slots exhausted (48 across live multi batches)");
  m->A.slot0 = slot0;
  int rc = VY_OK;
  if (cudaMemcpyToSymbol(c_groups, ps.data(), sizeof(Params) * (size_t)n, sizeof(Params) * (size_t)slot0) !=
      cudaSuccess)
    rc = fail(VY_ERR_CUDA, "cudaMemcpyToSymbol(c_groups)");
  if (!rc) rc = upload<unsigned long long>(&m->d_ctr, nullptr, 2);
  if (!rc && cudaMemset(m->d_ctr, 0, 16) != cudaSuccess) rc = fail(VY_ERR_CUDA, "memset");
  if (rc) {
    free_slots(slot0, n);
    cudaFree(m->d_ctr);
    return rc;
  }
  m->A.ctr = m->d_ctr;
  // geometry: as many warps per SM as shared memory allows (all sets staged per CTA)
  const vy_handle* h0 = hs[0];
  const int per_sm = h0->smem_per_sm;
  int best_w = 1, best_total = 0;
  for (int w = 1; w <= kMultiThreads / 32; ++w) {
    const int bytes = off + w * m->A.tile_bytes;
    if (bytes + 1024 > per_sm) break;
    const int total = (per_sm / (bytes + 1024)) * w;
    if (total >= best_total) {
      best_total = total;
      best_w = w;
    }
  }
  if (const char* ov = std::getenv("VY_WARPS_PER_CTA")) {
    const int w = std::atoi(ov);
    if (w >= 1 && w <= kMultiThreads / 32 && off + w * m->A.tile_bytes + 1024 <= per_sm) best_w = w;
  }
  m->warps = best_w;
  m->smem = off + best_w * m->A.tile_bytes;
  if (m->smem + 1024 > per_sm) return fail(VY_ERR_UNSUPPORTED, "groups too large for one shared-memory tile");
  auto* kern = mode == 1 ? k_step_multi<1> : mode == 2 ? k_step_multi<2> : mode == 3 ? k_step_multi<3> : k_step_multi<0>;
  VY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, m->smem));
  const unsigned resident = (unsigned)h0->num_sms * (unsigned)(per_sm / (m->smem + 1024));
  const unsigned want = (unsigned)((tiles + best_w - 1) / best_w);
  m->grid = want < resident ? want : resident;
  *out = m.release();
  return VY_OK;
}

int vy_multi_step_random(vy_multi* m, int64_t call, int64_t* call_counter, void* stream) {
  if (!m) return fail(VY_ERR_ARG, "null multi handle");
  vy::MultiArgs A = m->A;
  A.pol_call = call;
  A.pol_counter = call_counter;
  auto* kern = m->mode == 1 ? k_step_multi<1> : m->mode == 2 ? k_step_multi<2> : m->mode == 3 ? k_step_multi<3>
                                                                                                 : k_step_multi<0>;
  kern<<<m->grid, m->warps * 32, m->smem, (cudaStream_t)stream>>>(A);
  VY_CUDA(cudaGetLastError());
  ++m->launches;
  for (vy_handle* h : m->hs) h->last_mode = m->mode;
  return VY_OK;
}

int32_t vy_multi_info(vy_multi* m, int32_t* out4) {
  if (!m || !out4) return fail(VY_ERR_ARG, "null argument");
  out4[0] = m->mode;
  out4[1] = m->A.n_psets * 16 + m->A.n_ssets;
  out4[2] = m->warps;
  out4[3] = (int32_t)m->grid;
  return VY_OK;
}

int64_t vy_multi_launch_count(vy_multi* m) { return m ? m->launches : -1; }

int vy_multi_destroy(vy_multi* m) {
  if (!m) return VY_OK;
  free_slots(m->A.slot0, m->A.n_groups);
  cudaFree(m->d_ctr);
  delete m;
  return VY_OK;
}

}  // extern "C"
