/*
 * vy_oracle.c — CPU restatement of the reference step.  TEST INFRASTRUCTURE:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this; the product never does.
 *
 * Every block cites the reference line range it restates.  Arithmetic is
 * float64 with the reference's operation order and no FMA contraction (built
 * with -ffp-contract=off like setup.py:24), so results are bit-identical to
 * voltyard's compiled and pure-Python kernels.  Pinned against golden
 * trajectories generated from the reference itself (tests/golden/, made by
 * scripts/make_golden.py) and, when built, against oracle/_ref.
 */
#include "vy_oracle.h"

#include <math.h>
#include <pthread.h>
#include <string.h>

/* ---- splitmix64 streams: rng.py:20-115, _kernel.pyx:19-73 ---------------- */

#define SM_GOLDEN 0x9E3779B97F4A7C15ULL
#define SM_KEY0 0x8C2F9D1B6E4A5533ULL

static inline uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t sm_fold(uint64_t key, uint64_t part) { return sm_mix((key + SM_GOLDEN) ^ part); }

uint64_t vyo_stream_key2(uint64_t a, uint64_t b) { return sm_fold(sm_fold(SM_KEY0, a), b); }
uint64_t vyo_stream_key3(uint64_t a, uint64_t b, uint64_t c) { return sm_fold(vyo_stream_key2(a, b), c); }

static inline double sm_unit(uint64_t *st) {
  *st += SM_GOLDEN;
  return (double)(sm_mix(*st) >> 11) * (1.0 / 9007199254740992.0);
}

static inline int64_t sm_below(uint64_t *st, int64_t n) { /* Stream.randint rng.py:75-80 */
  int64_t k = (int64_t)(sm_unit(st) * (double)n);
  return k >= n ? n - 1 : k;
}

static int64_t sm_knuth(uint64_t *st, double lam) { /* rng.py:107-115 */
  const double thr = exp(-lam);
  double p = 1.0;
  int64_t k = 0;
  for (;;) {
    p *= sm_unit(st);
    if (p <= thr) return k;
    ++k;
  }
}

static int64_t sm_poisson(uint64_t *st, double lam) { /* rng.py:94-105 */
  if (lam <= 0.0) return 0;
  int64_t total = 0;
  while (lam > 32.0) {
    total += sm_knuth(st, 32.0);
    lam -= 32.0;
  }
  return total + sm_knuth(st, lam);
}

/* charge envelope, vehicles.py:22-35 / _kernel.pyx:76-79 */
static inline double envelope(double soc, double tau, double rbar) {
  return soc <= tau ? rbar : (1.0 - soc) * rbar / (1.0 - tau);
}

/* ---- per-env row view ----------------------------------------------------- */

typedef struct row {
  const vy_tables *t;
  int64_t n, ns, b;
  int8_t *occ, *pref;
  double *i_drawn, *soc, *de, *cap, *rbar, *tau, *rhat;
  int64_t *dtrem;
} row;

static row row_at(const vy_tables *t, vyo_state *s, int64_t b) {
  row r;
  const int64_t n = t->n_ports;
  r.t = t;
  r.n = n;
  r.ns = t->n_slots;
  r.b = b;
  r.occ = s->occ + b * n;
  r.pref = s->pref + b * n;
  r.i_drawn = s->i_drawn + b * n;
  r.soc = s->soc + b * n;
  r.de = s->de + b * n;
  r.cap = s->cap + b * n;
  r.rbar = s->rbar + b * n;
  r.tau = s->tau + b * n;
  r.rhat = s->rhat + b * n;
  r.dtrem = s->dtrem + b * n;
  return r;
}

static void vacate(row *r, int64_t i) { /* _kernel.pyx:263-273 */
  r->occ[i] = 0;
  r->pref[i] = 0;
  r->i_drawn[i] = r->soc[i] = r->de[i] = 0.0;
  r->cap[i] = r->rbar[i] = r->tau[i] = r->rhat[i] = 0.0;
  r->dtrem[i] = 0;
}

/* calendar position of a step: _kernel.pyx:289-291, 577-582 */
static void calendar(const vy_tables *t, int64_t tstep, int64_t day, int64_t *eff_day, int64_t *hour_idx) {
  const int64_t minutes = tstep * t->dt_min;
  *eff_day = (day + minutes / 1440) % t->n_days;
  *hour_idx = *eff_day * 24 + (minutes / 60) % 24;
}

/* observation row: _kernel.pyx:575-607, layout config.py:99-130 */
static void observe(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b) {
  row r = row_at(t, s, b);
  double *ob = o->obs + b * t->obs_len;
  const int64_t tstep = s->step[b], day = s->day[b];
  int64_t eff, hidx;
  calendar(t, tstep, day, &eff, &hidx);
  for (int64_t i = 0; i < r.n; ++i) {
    double *q = ob + 6 * i;
    q[0] = (double)r.occ[i];
    q[1] = r.i_drawn[i] / t->i_denom[i];
    q[2] = r.soc[i];
    q[3] = r.occ[i] ? r.de[i] / r.cap[i] : 0.0;
    q[4] = (double)r.dtrem[i] / (double)t->episode_steps;
    q[5] = (double)r.pref[i];
  }
  double *g = ob + 6 * r.n;
  g[0] = s->b_soc[b];
  g[1] = s->b_i[b] / t->b_idenom;
  g += 2;
  g[0] = t->buy[hidx];
  g[1] = t->sellg[hidx];
  g[2] = t->p_sell;
  g[3] = t->sin_t[tstep % t->steps_per_day];
  g[4] = t->cos_t[tstep % t->steps_per_day];
  g[5] = (double)t->weekday[eff];
  g[6] = (double)eff / 365.0;
  for (int64_t h = 0; h < t->horizon; ++h) {
    const int64_t fmin = (tstep + 1 + h) * t->dt_min;
    const int64_t fday = (day + fmin / 1440) % t->n_days;
    g[7 + h] = t->buy[fday * 24 + (fmin / 60) % 24];
  }
}

void vyo_reset_env(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b, int64_t episode) {
  /* _kernel.pyx:239-261 */
  uint64_t st = sm_fold(sm_fold(sm_fold(sm_fold(SM_KEY0, s->env_seed[b]), (uint64_t)episode), 0), 0);
  s->day[b] = sm_below(&st, t->n_days);
  s->step[b] = 0;
  s->episode[b] = episode;
  row r = row_at(t, s, b);
  for (int64_t i = 0; i < r.n; ++i) vacate(&r, i);
  if (t->battery_enabled) {
    s->b_soc[b] = t->b_init_soc;
    s->b_rhat[b] = envelope(t->b_init_soc, t->b_tau, t->b_rmax);
  } else {
    s->b_soc[b] = 0.0;
    s->b_rhat[b] = 0.0;
  }
  s->b_i[b] = 0.0;
  s->ep_profit[b] = s->ep_reward[b] = s->ep_missing[b] = s->ep_energy[b] = 0.0;
  s->ep_overtime[b] = s->ep_declined[b] = s->ep_departures[b] = 0;
  observe(t, s, o, b);
}

/* worst node overload on the requested currents: _kernel.pyx:611-624 */
static double overload(const vy_tables *t, const double *cur) {
  double worst = 0.0;
  for (int m = 0; m < t->n_nodes; ++m) {
    double acc = 0.0;
    for (int a = t->node_ptr[m]; a < t->node_ptr[m + 1]; ++a) acc += cur[t->node_leaf[a]];
    const double ld = acc > 0.0 ? acc / t->node_eta[m] : acc * t->node_eta[m];
    const double over = (ld >= 0.0 ? ld : -ld) - t->node_cap[m];
    if (over > worst) worst = over;
  }
  return worst;
}

/* proportional deepest-first rescale to a fixed point: _kernel.pyx:626-649 */
static void fit_tree(const vy_tables *t, double *cur) {
  for (int pass = 0; pass < t->max_passes; ++pass) {
    int moved = 0;
    for (int q = 0; q < t->n_nodes; ++q) {
      const int m = t->node_order[q];
      double acc = 0.0;
      for (int a = t->node_ptr[m]; a < t->node_ptr[m + 1]; ++a) acc += cur[t->node_leaf[a]];
      const double ld = acc > 0.0 ? acc / t->node_eta[m] : acc * t->node_eta[m];
      const double mag = ld >= 0.0 ? ld : -ld;
      if (mag > t->node_cap[m]) {
        const double f = t->node_cap[m] / mag;
        for (int a = t->node_ptr[m]; a < t->node_ptr[m + 1]; ++a) {
          const int j = t->node_leaf[a];
          const double v = cur[j] * f;
          if (v != cur[j]) {
            cur[j] = v;
            moved = 1;
          }
        }
      }
    }
    if (!moved) return;
  }
}

/* clip a target current to the envelope/port limits: _kernel.pyx:309-325 (ports)
 * and :329-345 (battery).  Charging uses rhat, discharging the mirrored envelope. */
static double clip_current(double target, double rhat, double soc, double tau, double rbar,
                           double volt, double imax_c, double imax_d) {
  if (target >= 0.0) {
    const double lim = 1000.0 * rhat / volt;
    double v = target;
    if (lim < v) v = lim;
    if (imax_c < v) v = imax_c;
    return v;
  }
  const double lim = 1000.0 * envelope(1.0 - soc, tau, rbar) / volt;
  double v = -target;
  if (lim < v) v = lim;
  if (imax_d < v) v = imax_d;
  return -v;
}

static void step_one(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b, const int64_t *actions) {
  row r = row_at(t, s, b);
  const int64_t n = r.n, ns = r.ns, na = n + 1;
  const int64_t *act = actions + b * na;
  const double kf = (double)t->k;
  const int64_t tstep = s->step[b];

  /* frame: _kernel.pyx:289-295 */
  int64_t eff, hidx;
  calendar(t, tstep, s->day[b], &eff, &hidx);
  const double p_buy = t->buy[hidx], p_sg = t->sellg[hidx];
  const double lam = t->lam[tstep % t->lam_len] * (t->weekday[eff] ? t->wk_scale : t->we_scale);

  /* phase 1, apply actions: _kernel.pyx:297-356 */
  double *cur = o->scratch + b * ns;
  for (int64_t i = 0; i < n; ++i) {
    if (!r.occ[i]) {
      cur[i] = 0.0;
      continue;
    }
    double target = r.i_drawn[i] + ((double)(act[i] - t->k) / kf) * t->imax_c[i];
    if (!t->allow_discharge && target < 0.0) target = 0.0;
    cur[i] = clip_current(target, r.rhat[i], r.soc[i], r.tau[i], r.rbar[i], t->volt[i], t->imax_c[i],
                          t->imax_d[i]);
  }
  if (t->battery_enabled) {
    const double target = s->b_i[b] + ((double)(act[n] - t->k) / kf) * t->b_imax;
    cur[n] = clip_current(target, s->b_rhat[b], s->b_soc[b], t->b_tau, t->b_rmax, t->b_volt, t->b_imax,
                          t->b_imax);
  }
  memcpy(o->i_att + b * ns, cur, sizeof(double) * ns);
  const double excess = overload(t, cur);
  fit_tree(t, cur);
  memcpy(o->i_used + b * ns, cur, sizeof(double) * ns);
  for (int64_t i = 0; i < n; ++i) r.i_drawn[i] = cur[i];
  if (t->battery_enabled) s->b_i[b] = cur[n];

  /* phase 2, charge: _kernel.pyx:358-424 (vehicles.py:137-208) */
  double e_net = 0.0, e_in = 0.0, e_out = 0.0;
  double *dl = o->delivered + b * n;
  for (int64_t i = 0; i < n; ++i) {
    double got = 0.0;
    if (r.occ[i]) {
      const double raw = t->dt_h * t->volt[i] * r.i_drawn[i] / 1000.0;
      got = raw;
      if (raw >= 0.0) {
        if (r.de[i] < got) got = r.de[i];
        const double room = r.cap[i] * (1.0 - r.soc[i]);
        if (room < got) got = room;
      } else {
        const double floor_ = -r.cap[i] * r.soc[i];
        if (got < floor_) got = floor_;
      }
      double soc = r.soc[i] + got / r.cap[i];
      soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
      r.soc[i] = soc;
      const double de = r.de[i] - got;
      r.de[i] = de < 0.0 ? 0.0 : de;
      r.rhat[i] = envelope(soc, r.tau[i], r.rbar[i]);
      e_net += got;
      if (got > 0.0)
        e_in += got / t->eta_c[i];
      else if (got < 0.0)
        e_out += got * t->eta_d[i];
    }
    dl[i] = got;
  }
  double e_b = 0.0, bgot = 0.0;
  if (t->battery_enabled) {
    bgot = t->dt_h * t->b_volt * s->b_i[b] / 1000.0;
    if (bgot >= 0.0) {
      const double room = t->b_cap * (1.0 - s->b_soc[b]);
      if (room < bgot) bgot = room;
    } else {
      const double floor_ = -t->b_cap * s->b_soc[b];
      if (bgot < floor_) bgot = floor_;
    }
    double soc = s->b_soc[b] + bgot / t->b_cap;
    soc = soc < 0.0 ? 0.0 : (soc > 1.0 ? 1.0 : soc);
    s->b_soc[b] = soc;
    s->b_rhat[b] = envelope(soc, t->b_tau, t->b_rmax);
    e_b = bgot > 0.0 ? bgot / t->b_eta_c : bgot * t->b_eta_d;
  }
  o->b_delivered[b] = bgot;
  for (int64_t i = 0; i < n; ++i)
    if (r.occ[i]) r.dtrem[i] -= 1;
  const double e_grid_net = e_in + e_out + e_b;

  /* phase 3, departures: _kernel.pyx:426-458 */
  int64_t nd = 0;
  double sat0 = 0.0, sat1 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!r.occ[i]) continue;
    const int8_t p = r.pref[i];
    const int64_t dt = r.dtrem[i];
    if (!((p == 0 && dt <= 0) || (p == 1 && r.de[i] == 0.0))) continue;
    const double missing = r.de[i];
    const int64_t over = dt < 0 ? -dt : 0, early = dt > 0 ? dt : 0;
    const int64_t at = b * n + nd;
    o->dep_port[at] = i;
    o->dep_missing[at] = missing;
    o->dep_overtime[at] = over;
    o->dep_early[at] = early;
    o->dep_pref[at] = p;
    o->dep_cap[at] = r.cap[i];
    o->dep_soc[at] = r.soc[i];
    if (p == 0)
      sat0 += missing;
    else
      sat1 += (double)over - t->beta * (double)early;
    s->ep_missing[b] += missing;
    s->ep_overtime[b] += over;
    s->ep_departures[b] += 1;
    vacate(&r, i);
    ++nd;
  }
  o->dep_n[b] = nd;

  /* phase 4, arrivals: _kernel.pyx:460-509 (data.py:188-219) */
  uint64_t st = sm_fold(sm_fold(sm_fold(sm_fold(SM_KEY0, s->env_seed[b]), (uint64_t)s->episode[b]), 1),
                        (uint64_t)tstep);
  const int64_t m = sm_poisson(&st, lam);
  int64_t nfree = 0;
  for (int64_t i = 0; i < n; ++i) nfree += r.occ[i] == 0;
  const int64_t admitted = m < nfree ? m : nfree;
  const int64_t declined = m - admitted;
  int64_t placed = 0;
  for (int64_t j = 0; j < m; ++j) {
    const double u = sm_unit(&st);
    int64_t car = t->n_cat - 1;
    for (int64_t e = 0; e < t->n_cat - 1; ++e)
      if (u < t->cat_cum[e]) {
        car = e;
        break;
      }
    const int64_t stay = t->stay_lo + sm_below(&st, t->stay_hi - t->stay_lo + 1);
    const double soc0 = t->soc_lo + sm_unit(&st) * (t->soc_hi - t->soc_lo);
    const double frac = t->frac_lo + sm_unit(&st) * (t->frac_hi - t->frac_lo);
    const int8_t pref = sm_unit(&st) < t->p_charge ? 1 : 0;
    if (placed >= admitted) continue;
    int64_t port = -1;
    for (int64_t q = 0; q < n; ++q)
      if (!r.occ[t->order[q]]) {
        port = t->order[q];
        break;
      }
    const double rb = t->kind[port] == 1 ? t->cat_rdc[car] : t->cat_rac[car];
    r.occ[port] = 1;
    r.i_drawn[port] = 0.0;
    r.soc[port] = soc0;
    r.cap[port] = t->cat_cap[car];
    r.rbar[port] = rb;
    r.tau[port] = t->cat_tau[car];
    r.de[port] = frac * t->cat_cap[car] * (1.0 - soc0);
    r.dtrem[port] = stay;
    r.pref[port] = pref;
    r.rhat[port] = envelope(soc0, t->cat_tau[car], rb);
    ++placed;
  }
  o->arrivals_m[b] = m;
  o->declined[b] = declined;
  s->ep_declined[b] += declined;

  /* reward: _kernel.pyx:511-551 */
  const double price = e_grid_net > 0.0 ? p_buy : p_sg;
  const double profit = t->p_sell * e_net - price * e_grid_net - t->c_dt;
  double *br = o->breakdown + b * 10;
  br[0] = profit;
  br[1] = excess;
  br[2] = sat0;
  br[3] = sat1;
  br[4] = t->has_moer ? t->moer[hidx] * e_grid_net : 0.0;
  br[5] = (double)declined;
  br[6] = e_b < 0.0 ? -e_b : 0.0;
  br[7] = e_out < 0.0 ? -e_out : 0.0;
  if (t->has_dgrid) {
    const double d = e_net - t->dgrid[hidx];
    br[8] = d >= 0.0 ? d : -d;
  } else {
    br[8] = 0.0;
  }
  double reward = profit;
  for (int c = 0; c < 8; ++c) reward -= t->alphas[c] * br[1 + c];
  br[9] = reward;
  o->reward[b] = reward;
  double *fl = o->flows + b * 5;
  fl[0] = e_net;
  fl[1] = e_in;
  fl[2] = e_out;
  fl[3] = e_b;
  fl[4] = e_grid_net;
  s->ep_profit[b] += profit;
  s->ep_reward[b] += reward;
  s->ep_energy[b] += e_net;

  /* advance: _kernel.pyx:553-571 */
  s->step[b] = tstep + 1;
  const int fin = tstep + 1 == t->episode_steps;
  o->done[b] = (int8_t)fin;
  int64_t tover = 0;
  if (fin) {
    for (int64_t i = 0; i < n; ++i)
      if (r.occ[i] && r.pref[i] == 1 && r.dtrem[i] < 0) tover += -r.dtrem[i];
    double *es = o->ep_stats + b * 8;
    es[0] = s->ep_profit[b];
    es[1] = s->ep_reward[b];
    es[2] = s->ep_missing[b];
    es[3] = (double)s->ep_overtime[b];
    es[4] = (double)s->ep_declined[b];
    es[5] = s->ep_energy[b];
    es[6] = (double)s->ep_departures[b];
    es[7] = (double)tover;
  }
  o->term_overtime[b] = tover;
  observe(t, s, o, b);
}

void vyo_step_range(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b0, int64_t b1,
                    const int64_t *actions) {
  for (int64_t b = b0; b < b1; ++b) step_one(t, s, o, b, actions);
}

typedef struct slice_job {
  const vy_tables *t;
  vyo_state *s;
  vyo_outs *o;
  int64_t b0, b1;
  const int64_t *a;
  int auto_reset;
} slice_job;

static void *run_slice(void *p) {
  slice_job *j = (slice_job *)p;
  vyo_step_range(j->t, j->s, j->o, j->b0, j->b1, j->a);
  /* engine.py:459-462: done rows start episode + 1 after the step (rows are
   * independent, so resetting inside the slice equals the engine's loop) */
  if (j->auto_reset)
    for (int64_t b = j->b0; b < j->b1; ++b)
      if (j->o->done[b]) vyo_reset_env(j->t, j->s, j->o, b, j->s->episode[b] + 1);
  return NULL;
}

static void step_slices(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B, const int64_t *actions,
                        int threads, int auto_reset) {
  if (threads < 1 || B < 2) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  slice_job jobs[256];
  for (int w = 0; w < threads; ++w) {
    jobs[w] = (slice_job){t, s, o, B * w / threads, B * (w + 1) / threads, actions, auto_reset};
    if (threads == 1)
      run_slice(&jobs[w]);
    else
      pthread_create(&th[w], NULL, run_slice, &jobs[w]);
  }
  if (threads > 1)
    for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
}

void vyo_step_parallel(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B, const int64_t *actions,
                       int threads) {
  step_slices(t, s, o, B, actions, threads, 0);
}

void vyo_step_parallel_autoreset(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B,
                                 const int64_t *actions, int threads) {
  step_slices(t, s, o, B, actions, threads, 1);
}

/* BatchEnv.reset over rows [0, B) (engine.py:414-424): episode 0 when `first`,
 * else each row's episode + 1; rows are independent, so slices run in parallel */
typedef struct reset_job {
  const vy_tables *t;
  vyo_state *s;
  vyo_outs *o;
  int64_t b0, b1;
  int first;
} reset_job;

static void *run_reset(void *p) {
  reset_job *j = (reset_job *)p;
  for (int64_t b = j->b0; b < j->b1; ++b) vyo_reset_env(j->t, j->s, j->o, b, j->first ? 0 : j->s->episode[b] + 1);
  return NULL;
}

void vyo_reset_parallel(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B, int first, int threads) {
  if (threads < 1 || B < 2) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  reset_job jobs[256];
  for (int w = 0; w < threads; ++w) {
    jobs[w] = (reset_job){t, s, o, B * w / threads, B * (w + 1) / threads, first};
    pthread_create(&th[w], NULL, run_reset, &jobs[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
}

/* RandomPolicy.actions over rows [0, B) on `threads` threads (row-independent streams) */
typedef struct pol_job {
  uint64_t *keys;
  int64_t b0, b1;
  int32_t n_slots, hi;
  int64_t *out;
} pol_job;

static void *run_pol(void *p) {
  pol_job *j = (pol_job *)p;
  vyo_random_actions(j->keys + j->b0, j->b1 - j->b0, j->n_slots, j->hi, j->out + j->b0 * j->n_slots);
  return NULL;
}

void vyo_random_actions_parallel(uint64_t *keys, int64_t B, int32_t n_slots, int32_t hi, int64_t *out,
                                 int threads) {
  if (threads < 1 || B < 2) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  pol_job jobs[256];
  for (int w = 0; w < threads; ++w) {
    jobs[w] = (pol_job){keys, B * w / threads, B * (w + 1) / threads, n_slots, hi, out};
    pthread_create(&th[w], NULL, run_pol, &jobs[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
}

void vyo_random_actions(uint64_t *keys, int64_t B, int32_t n_slots, int32_t hi, int64_t *out) {
  for (int64_t b = 0; b < B; ++b) {
    uint64_t st = keys[b];
    for (int32_t j = 0; j < n_slots; ++j) out[b * n_slots + j] = sm_below(&st, hi);
    keys[b] = st;
  }
}
