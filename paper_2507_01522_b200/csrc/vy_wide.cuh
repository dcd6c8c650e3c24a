// vy_wide.cuh — the small-batch rollout: one warp per environment, one lane
// per port.
//
// The tile kernels map one env to one thread, so a batch of B envs is B/32
// warps.  At the reference's own CPU-runnable size (config C1: 16 envs) that
// is ONE warp on one SM, and a step costs the full latency of ~7000 dependent
// instructions (~14 us).  Here a warp owns one env and lane j owns port j:
// the per-port work of a step (action, clip, charge, departure, obs) runs in
// parallel across the lanes, the port state stays in registers for all T
// steps, and only what the reference accumulates sequentially is serial — the
// node loads, energy flows and satisfaction penalties are summed over the
// ports in port order with warp shuffles (every lane computes the same sum,
// in the reference's order and roundings), and the per-env arithmetic
// (arrivals, reward, clocks) runs redundantly on every lane.  Semantics and
// operation order are tile_step's (vy_tile.cuh), so the outputs are
// bit-identical to k_rollout and to the reference.
//
// Lean configurations without a battery (Spec<1> / Spec<2>: any tree; node
// loads are summed from a per-warp shared copy of the currents, the energy
// flows from a shared copy of the per-port terms, broadcast reads in port
// order), at most 32 ports, float32 obs.  With `acts` the kernel is also the small-batch single
// step (T = 1) for caller-supplied uint8 actions (vy_step; the PPO rollout).
#pragma once

#include "vy_kernels.cuh"

namespace vy {

constexpr int kWideWarps = 8;  // warps (= envs) per CTA
constexpr int kWideScratch = 32 + 4 * 32;  // doubles of per-warp shared scratch

#ifdef VY_PPO_PROF  // phase stamps of the env step (scripts/probe_ppo_phases.py): CTA 0 thread 0, first 256 steps
__device__ unsigned long long g_env_stamp[256 * 16];
__device__ int g_env_t;
#define ENV_MARK(i)                                                                           \
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_env_t < 256) g_env_stamp[g_env_t * 16 + (i)] = clock64();
#define ENV_NEXT() \
  if (blockIdx.x == 0 && threadIdx.x == 0) ++g_env_t;
#else
#define ENV_MARK(i)
#define ENV_NEXT()
#endif

// _kernel.pyx:626-649 on a flat array of currents (lane 0 only; rare: a tree
// node over capacity).  Same values and pass structure as fit_tree.
__device__ __noinline__ void fit_tree_flat(const Params& P, TreeC tc, double* cur, int n, uint64_t clean) {
  const bool track = P.n_nodes <= 64;
  if (!track) clean = 0;
  for (int pass = 0; pass < P.max_passes; ++pass) {
    bool moved = false;
    for (int q = 0; q < P.n_nodes; ++q) {
      if ((clean >> q) & 1ull) continue;
      double cap, eta, rcp_eta;
      int lo, hi;
      tc.rec(q, cap, eta, rcp_eta, lo, hi);
      const int hp = hi < n ? hi : n;
      double s = 0.0;
      for (int j = lo; j < hp; ++j) s += cur[j];
      const double mag = fabs(node_load(s, eta, rcp_eta));
      bool mq = false;
      if (mag > cap) {
        const double f = cap / mag;
        for (int j = lo; j < hp; ++j) {
          const double v = cur[j] * f;
          if (v != cur[j]) {
            cur[j] = v;
            mq = true;
          }
        }
      }
      if (!track) {
        moved |= mq;
      } else if (mq) {
        moved = true;
        for (int r = 0; r < P.n_nodes; ++r) {
          double c2, e2, re2;
          int lo2, hi2;
          tc.rec(r, c2, e2, re2, lo2, hi2);
          if (lo2 < hi && lo < hi2) clean &= ~(1ull << r);
        }
      } else {
        clean |= 1ull << q;
      }
    }
    if (!moved) return;
  }
}

// One environment on one warp: lane j holds port j's constants and state in
// registers for as many steps as the caller runs; every lane also carries the
// env's scalars.  Shared by the rollout below and the fused PPO rollout
// (vy_ppo_rollout.cuh), which runs it on its env warps between policy passes.
template <int M>
struct WideEnv {
  static_assert(M == 1 || M == 2, "lean stations without a battery");
  double imax_c = 0.0, imax_d = 0.0, volt = 1.0, rcp_volt = 1.0, kindv = 0.0;
  double dtv = 0.0, eta_d = 1.0, eta_c = 1.0, rcp_eta_c = 1.0, i_denom = 1.0, rcp_i_denom = 1.0;
  double idr = 0.0, soc = 0.0, de = 0.0;
  int dt = 0;
  uint32_t mt = 0;
  EnvRegs E;
  int episode;
  uint64_t seed, nmask;
  double grid_lane;
  int64_t b;

  __device__ __forceinline__ void load(const Params& P, const PortC& pc, const double* dtab, int64_t b_, int lane) {
    b = b_;
    const int n = P.n_ports;
    if (lane < n) {
      double nodesv;
      pc.pair(lane, 0, imax_c, imax_d);
      pc.pair(lane, 1, volt, rcp_volt);
      pc.pair(lane, 2, kindv, nodesv);
      pc.pair(lane, 3, dtv, eta_d);
      pc.pair(lane, 4, eta_c, rcp_eta_c);
      pc.pair(lane, 5, i_denom, rcp_i_denom);
      const int64_t e = (int64_t)lane * P.ld + b;
      idr = P.st.port_i[e];
      soc = P.st.port_soc[e];
      de = P.st.port_de[e];
      dt = P.st.port_dtrem[e];
      mt = P.st.port_meta[e];
    }
    nmask = n == 64 ? ~0ull : ((1ull << n) - 1);
    load_env<M>(P, b, E);  // every lane: the env's scalars (broadcast loads)
    episode = P.st.episode[b];
    seed = P.st.env_seed[b];
    grid_lane = dtab[lane <= 2 * P.k ? lane : 0];  // (a-k)/k, one entry per lane (2k+1 <= 32)
  }

  __device__ __forceinline__ void store(const Params& P, int lane) const {
    if (lane < P.n_ports) {
      const int64_t e = (int64_t)lane * P.ld + b;
      P.st.port_i[e] = idr;
      P.st.port_soc[e] = soc;
      P.st.port_de[e] = de;
      P.st.port_dtrem[e] = (int16_t)dt;
      P.st.port_meta[e] = (uint8_t)mt;
    }
    if (lane == 0) {
      store_env<M>(P, b, E, true);
      P.st.episode[b] = episode;
    }
  }

  // One step with action `a` on this lane's port (P.k on lanes past the
  // ports): obs row -> orow (and, with kStage, a float copy -> srow), reward
  // and done -> element `rix` of P.out.reward / P.out.done.  cur_s / flow_s:
  // this warp's shared scratch (32 + 4 x 32 doubles).
  template <bool kStage>
  __device__ __forceinline__ void step(const Params& P, const Prof& prof, const TreeC& tc, int lane, int a,
                                       float* orow, float* srow, int64_t rix, double* cur_s, double* flow_s) {
    const unsigned FULL = 0xffffffffu;
    const int n = P.n_ports;
    const bool isport = lane < n;
    const int64_t ld = P.ld;
    ENV_MARK(0);
    const int tt = E.step;
    const Frame F = load_frame<M>(P, tt, E.day);
    // the obs globals of the state after this step, in flight during it (lanes 0..8 write them)
    ObsGlobals G{};
    if (lane < 9) G = load_obs_globals(P, tt + 1, E.day);
    const double d = __shfl_sync(FULL, grid_lane, a);

    // phase 1: apply actions (_kernel.pyx:297-356)
    const bool occ = mt & 1u;
    double c = 0.0;
    if (occ) {
      double tgt = idr + d * imax_c;
      if (!P.allow_discharge && tgt < 0.0) tgt = 0.0;
      const int pf = mt >> 2;
      c = clip_current(tgt, soc, prof.tau(pf), prof.omt(pf), prof.rcp_omt(pf),
                       kindv != 0.0 ? prof.r_dc(pf) : prof.r_ac(pf), volt, rcp_volt, imax_c, imax_d);
    }
    ENV_MARK(1);
    // tree: excess on the requested currents (_kernel.pyx:611-624), node loads in leaf order
    double excess = 0.0;
    uint64_t clean = 0;
    // node loads from a shared copy of the currents: lane q sums node q's
    // range in leaf order (the reference's order and roundings), so the
    // dependent chain is the largest range, not the sum of all ranges; the
    // excess is the max over the nodes' overloads (exact in any order) and
    // the within-capacity nodes a ballot
    if (isport) cur_s[lane] = c;
    __syncwarp();
    for (int q0 = 0; q0 < P.n_nodes; q0 += 32) {
      const int q = q0 + lane;
      double over = 0.0;
      bool ok = false;
      if (q < P.n_nodes) {
        double cap, eta, rcp_eta;
        int lo, hq;
        tc.rec(q, cap, eta, rcp_eta, lo, hq);
        const int hp = hq < n ? hq : n;
        double s = 0.0;
        for (int j = lo; j < hp; ++j) s += cur_s[j];
        over = fabs(node_load(s, eta, rcp_eta)) - cap;
        ok = !(over > 0.0);
      }
      if (over > excess) excess = over;
      const uint64_t bits = __ballot_sync(FULL, ok);
      if (q0 < 64) clean |= bits << q0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // warp max of the overloads (NaN never wins, as in the serial scan)
      const double x = __shfl_xor_sync(FULL, excess, o);
      if (x > excess) excess = x;
    }
    if (P.n_nodes > 64) clean = 0;  // fit_tree_flat tracks clean nodes only up to 64
    __syncwarp();
    ENV_MARK(9);
    if (excess > 0.0) {  // warp-uniform: every lane summed the same values
      if (isport) cur_s[lane] = c;
      __syncwarp();
      if (lane == 0) fit_tree_flat(P, tc, cur_s, n, clean);
      __syncwarp();
      if (isport) c = cur_s[lane];
      __syncwarp();
    }

    ENV_MARK(2);
    // phases 2+3: charge, dwell countdown, departures (_kernel.pyx:358-458)
    double got = 0.0, t_in = 0.0, t_out = 0.0, t_sat0 = 0.0, t_sat1 = 0.0, t_miss = 0.0;
    bool dep = false;
    int over = 0, t_over = 0;
    const int p = (mt >> 1) & 1u;
    if (occ) {
      const int pf = mt >> 2;
      const double raw = div_rcp(dtv * c, 1000.0, P.rcp_1000);
      double gc = raw;
      if (de < gc) gc = de;
      const double room = prof.cap(pf) * (1.0 - soc);
      if (room < gc) gc = room;
      const double fl = -prof.cap(pf) * soc;
      const double gd = raw < fl ? fl : raw;
      got = raw >= 0.0 ? gc : gd;
      soc = soc + div_rcp(got, prof.cap(pf), prof.rcp_cap(pf));
      soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
      de = de - got;
      de = de < 0.0 ? 0.0 : de;
      const double gin = eta_c == 1.0 ? got : div_rcp(got, eta_c, rcp_eta_c);
      t_in = got > 0.0 ? gin : 0.0;
      t_out = got < 0.0 ? got * eta_d : 0.0;
      dt -= 1;
      dep = (p == 0 && dt <= 0) || (p == 1 && de == 0.0);
      over = dt < 0 ? -dt : 0;
      const int early = dt > 0 ? dt : 0;
      if (dep) {
        t_miss = de;
        if (p == 0) t_sat0 = de;
        else t_sat1 = (double)over - P.beta * (double)early;
      }
      if (!dep && p == 1 && dt < 0) t_over = -dt;
    }
    ENV_MARK(3);
    // the reference's sequential sums over the ports, in port order, on every lane
    double e_net = 0.0, e_in = 0.0, e_out = 0.0;
    if (isport) {
      flow_s[4 * lane] = got;
      flow_s[4 * lane + 1] = t_in;
      flow_s[4 * lane + 2] = t_out;
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {  // broadcast reads: one 16-byte and one 8-byte load per port
      const double2 gi = *reinterpret_cast<const double2*>(flow_s + 4 * j);
      e_net += gi.x;
      e_in += gi.y;
      e_out += flow_s[4 * j + 2];
    }
    __syncwarp();
    ENV_MARK(4);
    double sat0 = 0.0, sat1 = 0.0;
    const unsigned depm = __ballot_sync(FULL, dep);
    if (depm) {
      for (int j = 0; j < n; ++j) {
        sat0 += __shfl_sync(FULL, t_sat0, j);
        sat1 += __shfl_sync(FULL, t_sat1, j);
        E.ep_missing += __shfl_sync(FULL, t_miss, j);
      }
      E.ep_overtime += __reduce_add_sync(FULL, dep ? over : 0);
      E.ep_departures += __popc(depm);
    }
    const bool last = tt + 1 == P.episode_steps;
    const int tover = last ? (int)__reduce_add_sync(FULL, (unsigned)t_over) : 0;
    if (dep) {
      mt = 0;
      c = soc = de = 0.0;
      dt = 0;
    }
    idr = c;
    uint64_t occm = (uint64_t)__ballot_sync(FULL, isport && (mt & 1u));

    ENV_MARK(5);
    // phase 4: arrivals (_kernel.pyx:460-509), drawn identically on every lane
    uint64_t st = fold(E.akey, (uint64_t)(int64_t)tt);
    int marr = 0;
    if (F.pfull >= 0) {
      for (int cc = 0; cc < F.pfull; ++cc) marr += knuth(st, P.thr32);
      marr += knuth(st, F.pthr);
    }
    const int nfree = n - __popcll(occm);
    const int admitted = marr < nfree ? marr : nfree;
    const int declined = marr - admitted;
    for (int j = 0; j < admitted; ++j) {
      const double u = unit(st);
      int car = P.n_cat - 1;
      for (int e = 0; e < P.n_cat - 1; ++e)
        if (u < prof.cum(e)) {
          car = e;
          break;
        }
      const int stay = P.stay_lo + below(st, P.stay_span);
      const double soc0 = P.soc_lo + unit(st) * P.soc_span;
      const double frac = P.frac_lo + unit(st) * P.frac_span;
      const uint32_t pref = unit(st) < P.p_charge ? 1u : 0u;
      const int port = __ffsll((long long)(~occm & nmask)) - 1;
      occm |= 1ull << port;
      if (lane == port) {
        mt = 1u | (pref << 1) | ((uint32_t)car << 2);
        idr = 0.0;
        soc = soc0;
        de = frac * prof.cap(car) * (1.0 - soc0);
        dt = stay;
      }
    }
    E.ep_declined += declined;

    ENV_MARK(6);
    // reward (_kernel.pyx:511-551), lean: no battery / carbon / demand terms
    const double e_b = 0.0;
    const double e_grid_net = e_in + e_out + e_b;
    const double price = e_grid_net > 0.0 ? F.p_buy : F.p_sg;
    const double profit = P.p_sell * e_net - price * e_grid_net - P.c_dt;
    double cpen[8];
    cpen[0] = excess;
    cpen[1] = sat0;
    cpen[2] = sat1;
    cpen[3] = 0.0;
    cpen[4] = (double)declined;
    cpen[5] = e_b < 0.0 ? -e_b : 0.0;
    cpen[6] = e_out < 0.0 ? -e_out : 0.0;
    cpen[7] = 0.0;
    double reward = profit;
#pragma unroll
    for (int q = 0; q < 8; ++q) reward -= P.alphas[q] * cpen[q];
    E.ep_profit += profit;
    E.ep_reward += reward;
    E.ep_energy += e_net;
    E.step = tt + 1;
    const bool done = tt + 1 == P.episode_steps;
    if (lane == 0) {
      if (done) {
        double* es = P.out.ep_stats;
        es[b] = E.ep_profit;
        es[ld + b] = E.ep_reward;
        es[2 * ld + b] = E.ep_missing;
        es[3 * ld + b] = (double)E.ep_overtime;
        es[4 * ld + b] = (double)E.ep_declined;
        es[5 * ld + b] = E.ep_energy;
        es[6 * ld + b] = (double)E.ep_departures;
        es[7 * ld + b] = (double)tover;
        P.out.term_overtime[b] = tover;
      }
      reinterpret_cast<float*>(P.out.reward)[rix] = (float)reward;
      P.out.done[rix] = done;
    }
    if (done) {  // in-kernel auto-reset: the obs row becomes the reset obs of episode + 1
      ++episode;
      reset_scalars(P, E, seed, episode, 0, false);
      mt = 0;
      idr = soc = de = 0.0;
      dt = 0;
    }

    ENV_MARK(7);
    // observation (_kernel.pyx:575-607): port j's six columns from lane j, the globals from lanes 0..8
    if (isport) {
      const bool o = mt & 1u;
      const double dec = div_rcp(de, prof.cap(mt >> 2), prof.rcp_cap(mt >> 2));
      const float v[6] = {o ? 1.0f : 0.0f, (float)div_rcp(idr, i_denom, rcp_i_denom), (float)soc,
                          o ? (float)dec : 0.0f, (float)div_rcp((double)dt, (double)P.episode_steps, P.rcp_ep),
                          (float)((mt >> 1) & 1u)};
      float* pr = orow + 6 * lane;
#pragma unroll
      for (int q = 0; q < 6; ++q) __stcs(pr + q, v[q]);
      if (kStage)
#pragma unroll
        for (int q = 0; q < 6; ++q) srow[6 * lane + q] = v[q];
    }
    if (lane < 9) {
      if (done) G = load_obs_globals(P, E.step, E.day);  // reset: the new episode's day
      const double v = lane == 0 ? E.b_soc
                       : lane == 1 ? div_rcp(E.b_i, P.b_idenom, P.b_rcp_idenom)
                       : lane == 2 ? G.buy
                       : lane == 3 ? G.sellg
                       : lane == 4 ? P.p_sell
                       : lane == 5 ? G.sinv
                       : lane == 6 ? G.cosv
                       : lane == 7 ? G.wk
                                   : G.dayf;
      __stcs(orow + 6 * n + lane, (float)v);
      if (kStage) srow[6 * n + lane] = (float)v;
    }
    ENV_MARK(8);
    ENV_NEXT();
  }
};

template <int M>
__global__ void __launch_bounds__(32 * kWideWarps) k_rollout_wide(const __grid_constant__ Params P, int T_steps,
                                                                  uint64_t policy_seed, int64_t index0, int64_t call0,
                                                                  int64_t obs_stride, int64_t rew_stride,
                                                                  const uint8_t* __restrict__ acts) {
  Prof prof;
  PortC pc;
  TreeC tc;
  const double* dtab;
  stage_tables(P, prof, dtab, pc, tc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * kWideWarps + warp;
  if (b >= P.B) return;
  const int n = P.n_ports, OL = P.obs_len;
  // per-warp scratch: the ports' currents (node loads, rescale) and their
  // energy-flow terms {got, in, out, -} (the sequential flow sums)
  double* cur_s = reinterpret_cast<double*>(vy_smem + tables_bytes(P.n_profiles, P.k, P.n_ports, P.n_nodes)) +
                  warp * kWideScratch;
  double* flow_s = cur_s + 32;
  WideEnv<M> env;
  env.load(P, pc, dtab, b, lane);
  const uint64_t pkey = fold(fold(fold(kKey0, policy_seed), (uint64_t)(index0 + b)), 2);
  const int ns = n + 1, hi = 2 * P.k + 1, hi_a = 2 * P.k;

  for (int t = 0; t < T_steps; ++t) {
    // slot j's action on lane j: RandomPolicy (policies.py:51-73), or the
    // caller's uint8 rows [B][n+1] (vy_step: one step, acts != null)
    int a = P.k;
    if (lane < n) {
      if (acts) {
        a = acts[b * ns + lane];
        if (a > hi_a) {  // out of range: clamped and flagged (the lazy error word, engine.py:440-442)
          atomicOr(P.err, 1u);
          a = hi_a;
        }
      } else {
        a = policy_action(pkey, (uint64_t)(call0 + t) * (uint64_t)ns + lane + 1, hi);
      }
    }
    if (acts && lane == 0 && acts[b * ns + n] > hi_a) atomicOr(P.err, 1u);  // the battery slot is validated too
    float* orow = reinterpret_cast<float*>(P.out.obs) + t * obs_stride + b * OL;
    env.template step<false>(P, prof, tc, lane, a, orow, nullptr, t * rew_stride + b, cur_s, flow_s);
  }
  env.store(P, lane);
}

}  // namespace vy
