// vy_step.cuh — the fused environment transition, one thread per environment.
//
// Semantics: voltyard/backends/_kernel.pyx:239-649 (== pykernel.py:30-429),
// restated for the GPU.  Mapping: thread b owns env b for the whole step; its
// ports live in registers (the template capacity NP is a compile-time port
// count, so every per-port loop is unrolled and every port array is register
// resident).  All continuous arithmetic is float64 in the reference's exact
// operation order and the translation unit is built with --fmad=false, so
// each env's trajectory is bit-identical to the reference's compiled kernel.
// Sums the reference accumulates sequentially (tree node loads, energy flows,
// satisfaction penalties) are accumulated sequentially here too — that is
// why the mapping is thread-per-env rather than lane-per-port: a warp-shuffle
// tree reduction would reassociate float64 additions.
#pragma once

#include "vy_device.cuh"

namespace vy {

template <int NP>
struct Env {
  double idr[NP], soc[NP], de[NP];
  int dtrem[NP];
  uint32_t meta[NP];  // bit0 occupied, bit1 preference, bits2..7 profile id
  int step, day;
  uint64_t akey;
  double b_i, b_soc;
  double ep_profit, ep_reward, ep_missing, ep_energy;
  int ep_overtime, ep_declined, ep_departures;
};

template <int NP>
__device__ __forceinline__ void load_env(const Params<NP>& P, int64_t b, Env<NP>& E) {
  const vy_state& s = P.st;
  const int64_t ld = P.ld;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    if (i < P.n_ports) {
      E.idr[i] = s.port_i[i * ld + b];
      E.soc[i] = s.port_soc[i * ld + b];
      E.de[i] = s.port_de[i * ld + b];
      E.dtrem[i] = s.port_dtrem[i * ld + b];
      E.meta[i] = s.port_meta[i * ld + b];
    } else {
      E.idr[i] = E.soc[i] = E.de[i] = 0.0;
      E.dtrem[i] = 0;
      E.meta[i] = 0;
    }
  }
  E.step = s.step[b];
  E.day = s.day[b];
  E.akey = s.akey[b];
  if (P.battery) {
    E.b_i = s.b_i[b];
    E.b_soc = s.b_soc[b];
  } else {
    E.b_i = E.b_soc = 0.0;
  }
  E.ep_profit = s.ep_profit[b];
  E.ep_reward = s.ep_reward[b];
  E.ep_missing = s.ep_missing[b];
  E.ep_energy = s.ep_energy[b];
  E.ep_overtime = s.ep_overtime[b];
  E.ep_declined = s.ep_declined[b];
  E.ep_departures = s.ep_departures[b];
}

template <int NP>
__device__ __forceinline__ void store_env(const Params<NP>& P, int64_t b, const Env<NP>& E, bool reset_too) {
  const vy_state& s = P.st;
  const int64_t ld = P.ld;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    if (i < P.n_ports) {
      s.port_i[i * ld + b] = E.idr[i];
      s.port_soc[i * ld + b] = E.soc[i];
      s.port_de[i * ld + b] = E.de[i];
      s.port_dtrem[i * ld + b] = (int16_t)E.dtrem[i];
      s.port_meta[i * ld + b] = (uint8_t)E.meta[i];
    }
  }
  s.step[b] = E.step;
  if (P.battery) {
    s.b_i[b] = E.b_i;
    s.b_soc[b] = E.b_soc;
  }
  s.ep_profit[b] = E.ep_profit;
  s.ep_reward[b] = E.ep_reward;
  s.ep_missing[b] = E.ep_missing;
  s.ep_energy[b] = E.ep_energy;
  s.ep_overtime[b] = E.ep_overtime;
  s.ep_declined[b] = E.ep_declined;
  s.ep_departures[b] = E.ep_departures;
  if (reset_too) {
    s.day[b] = E.day;
    s.akey[b] = E.akey;
  }
}

// charge envelope (vehicles.py:22-35); omt = 1 - tau precomputed with identical rounding
__device__ __forceinline__ double envelope(double soc, double tau, double omt, double rbar) {
  return soc <= tau ? rbar : (1.0 - soc) * rbar / omt;
}

// Clip a requested current (_kernel.pyx:309-325 for ports, :329-345 battery).
// Charging is bounded by rhat = envelope(soc) (the value the reference stores,
// _kernel.pyx:389/505), discharging by envelope(1 - soc); both written as one
// select-based path so a warp does not diverge on the sign of the request.
__device__ __forceinline__ double clip_current(double tgt, double soc, double tau, double omt, double rbar,
                                               double volt, double imax_c, double imax_d) {
  const bool chg = tgt >= 0.0;
  const double s = chg ? soc : 1.0 - soc;
  const double r = envelope(s, tau, omt, rbar);
  const double lim = 1000.0 * r / volt;
  double v = chg ? tgt : -tgt;
  if (lim < v) v = lim;
  const double pm = chg ? imax_c : imax_d;
  if (pm < v) v = pm;
  return chg ? v : -v;
}

// reset_env (_kernel.pyx:239-261) on registers; episode = new episode number.
template <int NP>
__device__ __forceinline__ void reset_regs(const Params<NP>& P, Env<NP>& E, uint64_t seed, int episode,
                                           const int32_t* inj_day, int64_t b) {
  uint64_t st = fold(fold(fold(fold(kKey0, seed), (uint64_t)(int64_t)episode), 0), 0);
  E.day = inj_day ? inj_day[b] : below(st, P.n_days);
  E.step = 0;
  E.akey = fold(fold(fold(kKey0, seed), (uint64_t)(int64_t)episode), 1);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    E.idr[i] = E.soc[i] = E.de[i] = 0.0;
    E.dtrem[i] = 0;
    E.meta[i] = 0;
  }
  E.b_soc = P.battery ? P.b_init_soc : 0.0;
  E.b_i = 0.0;
  E.ep_profit = E.ep_reward = E.ep_missing = E.ep_energy = 0.0;
  E.ep_overtime = E.ep_declined = E.ep_departures = 0;
}

// tree node load over slots [lo, hi): ports in leaf order, then the battery slot
template <int NP>
__device__ __forceinline__ double node_sum(const Params<NP>& P, const double (&cur)[NP], double cb, int m) {
  const int lo = P.node_lo[m], hi = P.node_hi[m];
  const int hp = hi < P.n_ports ? hi : P.n_ports;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < NP; ++j)
    if (j >= lo && j < hp) s += cur[j];
  if (P.battery && lo <= P.n_ports && P.n_ports < hi) s += cb;
  return s;
}

__device__ __forceinline__ double node_load(double s, double eta) {
  // x / 1.0 == x and x * 1.0 == x exactly, so unit efficiencies skip the divide
  if (s > 0.0) return eta == 1.0 ? s : s / eta;
  return s * eta;
}

template <int NP>
__device__ __forceinline__ void fit_tree(const Params<NP>& P, double (&cur)[NP], double& cb) {
  // _kernel.pyx:626-649: deepest-first proportional scaling to a fixed point
  for (int pass = 0; pass < P.max_passes; ++pass) {
    bool moved = false;
    for (int q = 0; q < P.n_nodes; ++q) {
      const int m = P.node_order[q];
      const double mag = fabs(node_load(node_sum(P, cur, cb, m), P.node_eta[m]));
      if (mag > P.node_cap[m]) {
        const double f = P.node_cap[m] / mag;
        const int lo = P.node_lo[m], hi = P.node_hi[m];
        const int hp = hi < P.n_ports ? hi : P.n_ports;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          if (j >= lo && j < hp) {
            const double v = cur[j] * f;
            if (v != cur[j]) {
              cur[j] = v;
              moved = true;
            }
          }
        }
        if (P.battery && lo <= P.n_ports && P.n_ports < hi) {
          const double v = cb * f;
          if (v != cb) {
            cb = v;
            moved = true;
          }
        }
      }
    }
    if (!moved) return;
  }
}

struct StepResult {
  double reward;
  bool done;
};

// One transition of one env (_kernel.pyx:283-571).  `act(slot)` returns the
// action index of a slot; `b` is the env index (for info / injected draws).
template <int NP, class Act>
__device__ __forceinline__ StepResult step_env(const Params<NP>& P, const Profile* __restrict__ prof,
                                               const double* __restrict__ dtab, Env<NP>& E, int64_t b, Act act) {
  const int n = P.n_ports;
  const int64_t ld = P.ld;
  const bool info = P.flags & VY_F_INFOS;
  const vy_outputs& O = P.out;
  const int t = E.step;

  // frame (_kernel.pyx:289-295)
  const int64_t minutes = (int64_t)t * P.dt_min;
  const int eff_day = (int)(((int64_t)E.day + minutes / 1440) % P.n_days);
  const int hidx = eff_day * 24 + (int)((minutes / 60) % 24);
  const double p_buy = __ldg(P.buy + hidx), p_sg = __ldg(P.sellg + hidx);
  const int lam_idx = (__ldg(P.weekday + eff_day) ? 0 : P.lam_len) + t % P.lam_len;

  // phase 1: apply actions (_kernel.pyx:297-356)
  const int hi_a = 2 * P.k;
  auto delta_of = [&](int a) -> double {
    if (a < 0 || a > hi_a) {
      atomicOr(P.err, 1u);
      a = a < 0 ? 0 : hi_a;
    }
    return dtab ? dtab[a] : (double)(a - P.k) / (double)P.k;
  };
  double cur[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    cur[i] = 0.0;
    if (i < n) {
      const double d = delta_of(act(i));
      if (E.meta[i] & 1u) {
        double tgt = E.idr[i] + d * P.imax_c[i];
        if (!P.allow_discharge && tgt < 0.0) tgt = 0.0;
        const Profile& pr = prof[E.meta[i] >> 2];
        cur[i] = clip_current(tgt, E.soc[i], pr.tau, pr.omt, P.kind[i] ? pr.r_dc : pr.r_ac, P.volt[i],
                              P.imax_c[i], P.imax_d[i]);
      }
    }
  }
  double cb = 0.0;
  {
    // the battery slot is validated even when the battery is disabled (engine.py:440-442)
    const double d = delta_of(act(n));
    if (P.battery) {
      const double tgt = E.b_i + d * P.b_imax;
      cb = clip_current(tgt, E.b_soc, P.b_tau, P.b_omt, P.b_rmax, P.b_volt, P.b_imax, P.b_imax);
    }
  }
  if (info) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
      if (i < n) O.i_att[i * ld + b] = cur[i];
    if (P.battery) O.i_att[n * ld + b] = cb;
  }
  // tree: excess on the requested currents (_kernel.pyx:611-624), then rescale
  double excess = 0.0;
  for (int m = 0; m < P.n_nodes; ++m) {
    const double over = fabs(node_load(node_sum(P, cur, cb, m), P.node_eta[m])) - P.node_cap[m];
    if (over > excess) excess = over;
  }
  // no node over capacity => the first rescale pass changes nothing and returns
  if (excess > 0.0) fit_tree(P, cur, cb);
  if (info) {
#pragma unroll
    for (int i = 0; i < NP; ++i)
      if (i < n) O.i_used[i * ld + b] = cur[i];
    if (P.battery) O.i_used[n * ld + b] = cb;
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) E.idr[i] = cur[i];
  if (P.battery) E.b_i = cb;

  // phase 2: charge (_kernel.pyx:358-424)
  double e_net = 0.0, e_in = 0.0, e_out = 0.0;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double got = 0.0;
    if (i < n && (E.meta[i] & 1u)) {
      const Profile& pr = prof[E.meta[i] >> 2];
      const double raw = P.dtv[i] * E.idr[i] / 1000.0;
      got = raw;
      if (raw >= 0.0) {
        if (E.de[i] < got) got = E.de[i];
        const double room = pr.cap * (1.0 - E.soc[i]);
        if (room < got) got = room;
      } else {
        const double fl = -pr.cap * E.soc[i];
        if (got < fl) got = fl;
      }
      double soc = E.soc[i] + got / pr.cap;
      soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
      E.soc[i] = soc;
      const double de = E.de[i] - got;
      E.de[i] = de < 0.0 ? 0.0 : de;
      e_net += got;
      if (got > 0.0)
        e_in += P.eta_c[i] == 1.0 ? got : got / P.eta_c[i];
      else if (got < 0.0)
        e_out += got * P.eta_d[i];
    }
    if (info && i < n) O.delivered[i * ld + b] = got;
  }
  double e_b = 0.0, bgot = 0.0;
  if (P.battery) {
    bgot = P.b_dtv * E.b_i / 1000.0;
    if (bgot >= 0.0) {
      const double room = P.b_cap * (1.0 - E.b_soc);
      if (room < bgot) bgot = room;
    } else {
      const double fl = -P.b_cap * E.b_soc;
      if (bgot < fl) bgot = fl;
    }
    double soc = E.b_soc + bgot / P.b_cap;
    E.b_soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
    e_b = bgot > 0.0 ? bgot / P.b_eta_c : bgot * P.b_eta_d;
  }
  if (info) O.b_delivered[b] = bgot;
#pragma unroll
  for (int i = 0; i < NP; ++i)
    if (E.meta[i] & 1u) E.dtrem[i] -= 1;
  const double e_grid_net = e_in + e_out + e_b;

  // phase 3: departures, in port order (_kernel.pyx:426-458)
  int nd = 0;
  double sat0 = 0.0, sat1 = 0.0;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const uint32_t mt = E.meta[i];
    if (!(mt & 1u)) continue;
    const int p = (mt >> 1) & 1u;
    const int dt = E.dtrem[i];
    if (!((p == 0 && dt <= 0) || (p == 1 && E.de[i] == 0.0))) continue;
    const double missing = E.de[i];
    const int over = dt < 0 ? -dt : 0, early = dt > 0 ? dt : 0;
    if (info) {
      const int64_t at = (int64_t)nd * ld + b;
      O.dep_port[at] = i;
      O.dep_missing[at] = missing;
      O.dep_overtime[at] = over;
      O.dep_early[at] = early;
      O.dep_pref[at] = p;
      O.dep_cap[at] = prof[mt >> 2].cap;
      O.dep_soc[at] = E.soc[i];
    }
    if (p == 0)
      sat0 += missing;
    else
      sat1 += (double)over - P.beta * (double)early;
    E.ep_missing += missing;
    E.ep_overtime += over;
    E.ep_departures += 1;
    E.meta[i] = 0;
    E.idr[i] = E.soc[i] = E.de[i] = 0.0;
    E.dtrem[i] = 0;
    ++nd;
  }
  if (info) O.dep_n[b] = nd;

  // phase 4: arrivals (_kernel.pyx:460-509); draws of Stream(key4(seed, ep, 1, t))
  uint64_t st = fold(E.akey, (uint64_t)(int64_t)t);
  const bool inj = P.flags & VY_F_INJECT;
  int m = 0;
  int64_t inj0 = 0;
  if (inj) {
    inj0 = P.inj.off[b];
    m = P.inj.off[b + 1] - (int)inj0;
  } else {
    const int full = __ldg(P.pois_full + lam_idx);
    if (full >= 0) {
      for (int c = 0; c < full; ++c) m += knuth(st, P.thr32);
      m += knuth(st, __ldg(P.pois_thr + lam_idx));
    }
  }
  uint64_t occm = 0;
#pragma unroll
  for (int i = 0; i < NP; ++i)
    if (E.meta[i] & 1u) occm |= 1ull << i;
  const int nfree = n - __popcll(occm);
  const int admitted = m < nfree ? m : nfree;
  const int declined = m - admitted;
  for (int j = 0; j < m; ++j) {
    int car, stay;
    double soc0, frac;
    uint32_t pref;
    if (inj) {
      car = P.inj.profile[inj0 + j];
      stay = P.inj.stay[inj0 + j];
      soc0 = P.inj.soc0[inj0 + j];
      frac = P.inj.frac[inj0 + j];
      pref = P.inj.pref[inj0 + j] ? 1u : 0u;
    } else {
      const double u = unit(st);
      car = P.n_cat - 1;
      for (int e = 0; e < P.n_cat - 1; ++e)
        if (u < __ldg(P.cat_cum + e)) {
          car = e;
          break;
        }
      stay = P.stay_lo + below(st, P.stay_span);
      soc0 = P.soc_lo + unit(st) * P.soc_span;
      frac = P.frac_lo + unit(st) * P.frac_span;
      pref = unit(st) < P.p_charge ? 1u : 0u;
    }
    if (j >= admitted) continue;
    int port;
    const uint64_t freem = ~occm & (n == 64 ? ~0ull : ((1ull << n) - 1));
    if (P.order_identity) {
      port = __ffsll((long long)freem) - 1;
    } else {
      port = 0;
      for (int q = 0; q < n; ++q)
        if ((freem >> P.order[q]) & 1ull) {
          port = P.order[q];
          break;
        }
    }
    occm |= 1ull << port;
    const double de0 = frac * prof[car].cap * (1.0 - soc0);
    const uint32_t mt = 1u | (pref << 1) | ((uint32_t)car << 2);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      if (i == port) {
        E.meta[i] = mt;
        E.idr[i] = 0.0;
        E.soc[i] = soc0;
        E.de[i] = de0;
        E.dtrem[i] = stay;
      }
    }
  }
  E.ep_declined += declined;
  if (info) {
    O.arrivals_m[b] = m;
    O.declined[b] = declined;
  }

  // reward (_kernel.pyx:511-551)
  const double price = e_grid_net > 0.0 ? p_buy : p_sg;
  const double profit = P.p_sell * e_net - price * e_grid_net - P.c_dt;
  double c[8];
  c[0] = excess;
  c[1] = sat0;
  c[2] = sat1;
  c[3] = P.has_moer ? __ldg(P.moer + hidx) * e_grid_net : 0.0;
  c[4] = (double)declined;
  c[5] = e_b < 0.0 ? -e_b : 0.0;
  c[6] = e_out < 0.0 ? -e_out : 0.0;
  if (P.has_dgrid) {
    const double d = e_net - __ldg(P.dgrid + hidx);
    c[7] = d >= 0.0 ? d : -d;
  } else {
    c[7] = 0.0;
  }
  double reward = profit;
#pragma unroll
  for (int q = 0; q < 8; ++q) reward -= P.alphas[q] * c[q];
  if (info) {
    O.breakdown[b] = profit;
#pragma unroll
    for (int q = 0; q < 8; ++q) O.breakdown[(q + 1) * ld + b] = c[q];
    O.breakdown[9 * ld + b] = reward;
    O.flows[b] = e_net;
    O.flows[ld + b] = e_in;
    O.flows[2 * ld + b] = e_out;
    O.flows[3 * ld + b] = e_b;
    O.flows[4 * ld + b] = e_grid_net;
  }
  E.ep_profit += profit;
  E.ep_reward += reward;
  E.ep_energy += e_net;

  // advance (_kernel.pyx:553-570)
  E.step = t + 1;
  const bool done = t + 1 == P.episode_steps;
  if (done || info) {
    int tover = 0;
    if (done) {
#pragma unroll
      for (int i = 0; i < NP; ++i)
        if ((E.meta[i] & 3u) == 3u && E.dtrem[i] < 0) tover += -E.dtrem[i];
      double* es = O.ep_stats;
      es[b] = E.ep_profit;
      es[ld + b] = E.ep_reward;
      es[2 * ld + b] = E.ep_missing;
      es[3 * ld + b] = (double)E.ep_overtime;
      es[4 * ld + b] = (double)E.ep_declined;
      es[5 * ld + b] = E.ep_energy;
      es[6 * ld + b] = (double)E.ep_departures;
      es[7 * ld + b] = (double)tover;
    }
    O.term_overtime[b] = tover;
  }
  return {reward, done};
}

// Observation row (_kernel.pyx:575-607; layout config.py:99-130).  T is float
// (rounded once from the exact float64 value) or double.
template <int NP, typename T>
__device__ __forceinline__ void write_obs(const Params<NP>& P, const Profile* __restrict__ prof,
                                          const Env<NP>& E, T* __restrict__ row) {
  const int n = P.n_ports;
  const int t = E.step;
  const int64_t minutes = (int64_t)t * P.dt_min;
  const int eff_day = (int)(((int64_t)E.day + minutes / 1440) % P.n_days);
  const int hidx = eff_day * 24 + (int)((minutes / 60) % 24);
  const int sod = t % P.steps_per_day;
  const double ep_len = (double)P.episode_steps;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    if (i < n) {
      const uint32_t mt = E.meta[i];
      const bool occ = mt & 1u;
      const double idr = E.idr[i], de = E.de[i];
      T* q = row + 6 * i;
      q[0] = (T)(occ ? 1.0 : 0.0);
      q[1] = (T)(idr == 0.0 ? idr : idr / P.i_denom[i]);
      q[2] = (T)E.soc[i];
      q[3] = (T)(occ ? (de == 0.0 ? de : de / prof[mt >> 2].cap) : 0.0);
      q[4] = (T)(E.dtrem[i] == 0 ? 0.0 : (double)E.dtrem[i] / ep_len);
      q[5] = (T)(double)((mt >> 1) & 1u);
    }
  }
  T* g = row + 6 * n;
  g[0] = (T)E.b_soc;
  g[1] = (T)(E.b_i == 0.0 ? E.b_i : E.b_i / P.b_idenom);
  g[2] = (T)__ldg(P.buy + hidx);
  g[3] = (T)__ldg(P.sellg + hidx);
  g[4] = (T)P.p_sell;
  g[5] = (T)__ldg(P.sin_t + sod);
  g[6] = (T)__ldg(P.cos_t + sod);
  g[7] = (T)(double)__ldg(P.weekday + eff_day);
  g[8] = (T)((double)eff_day / 365.0);
  for (int h = 0; h < P.horizon; ++h) {
    const int64_t fmin = (int64_t)(t + 1 + h) * P.dt_min;
    const int64_t fday = ((int64_t)E.day + fmin / 1440) % P.n_days;
    g[9 + h] = (T)__ldg(P.buy + fday * 24 + (fmin / 60) % 24);
  }
}

}  // namespace vy
