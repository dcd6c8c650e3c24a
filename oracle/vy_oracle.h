/*
 * vy_oracle.h — CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * A plain-C restatement of the reference step (voltyard/backends/_kernel.pyx
 * and its Python twin pykernel.py), used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the *checker*.  Nothing in the product
 * path may link or call it.
 *
 * State and outputs use the reference's own layout (row-major [B][n],
 * float64 / int64 / int8; engine.py:221-336) so the oracle is a literal
 * drop-in for CySimCore and can be cross-checked against the real compiled
 * reference (oracle/_ref) on identical arrays.
 */
#ifndef VY_ORACLE_H
#define VY_ORACLE_H

#include <stdint.h>
#include "../include/voltyard_b200.h"

typedef struct vyo_state {
  int8_t *occ, *pref;                                    /* [B][N] */
  double *i_drawn, *soc, *de, *cap, *rbar, *tau, *rhat;  /* [B][N] */
  int64_t *dtrem;                                        /* [B][N] */
  double *b_i, *b_soc, *b_rhat;                          /* [B]    */
  int64_t *step, *day, *episode;                         /* [B]    */
  uint64_t *env_seed;                                    /* [B]    */
  double *ep_profit, *ep_reward, *ep_missing, *ep_energy;/* [B]    */
  int64_t *ep_overtime, *ep_declined, *ep_departures;    /* [B]    */
} vyo_state;

typedef struct vyo_outs {
  double *obs;          /* [B][obs_len] */
  double *reward;       /* [B] */
  int8_t *done;         /* [B] */
  double *breakdown;    /* [B][10] */
  double *flows;        /* [B][5] */
  int64_t *declined, *arrivals_m, *dep_n; /* [B] */
  int64_t *dep_port;    /* [B][N] */
  double *dep_missing;  /* [B][N] */
  int64_t *dep_overtime, *dep_early, *dep_pref; /* [B][N] */
  double *dep_cap, *dep_soc; /* [B][N] */
  int64_t *term_overtime; /* [B] */
  double *ep_stats;     /* [B][8] */
  double *i_att, *i_used; /* [B][n_slots] */
  double *delivered;    /* [B][N] */
  double *b_delivered;  /* [B] */
  double *scratch;      /* [B][n_slots] */
} vyo_outs;

void vyo_reset_env(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b, int64_t episode);
void vyo_step_range(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t b0, int64_t b1,
                    const int64_t *actions /* [B][N+1] */);
/* Multi-threaded step over [0, B) with `threads` pthreads (the reference's
 * worker split, engine.py:446-456); results are identical for any count. */
void vyo_step_parallel(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B,
                       const int64_t *actions, int threads);
/* The same with the engine's auto-reset of done rows (episode + 1,
 * engine.py:459-462) done inside each slice. */
void vyo_step_parallel_autoreset(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B,
                                 const int64_t *actions, int threads);
/* BatchEnv.reset of rows [0, B): episode 0 if `first`, else episode + 1. */
void vyo_reset_parallel(const vy_tables *t, vyo_state *s, vyo_outs *o, int64_t B, int first, int threads);
/* RandomPolicy.actions for rows [0,B): keys[b] is the row's stream state,
 * advanced in place (policies.py:69-73, rng.py:154-170). */
void vyo_random_actions(uint64_t *keys, int64_t B, int32_t n_slots, int32_t hi, int64_t *out);
void vyo_random_actions_parallel(uint64_t *keys, int64_t B, int32_t n_slots, int32_t hi, int64_t *out,
                                 int threads);
uint64_t vyo_stream_key2(uint64_t a, uint64_t b);
uint64_t vyo_stream_key3(uint64_t a, uint64_t b, uint64_t c);

#endif
