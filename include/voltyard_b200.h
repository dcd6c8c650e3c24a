/*
 * voltyard_b200.h — C ABI of the B200-native vectorised charging-station step.
 *
 * This is the drop-in boundary for the reference's batched rollout path.  The
 * reference binds its stepping core through a Python plugin registry:
 *
 *   make_core(tables, states, outs, backend)        backends/__init__.py:43-47
 *   core.reset_env(b, episode)                      backends/_kernel.pyx:239-261
 *   core.step_range(b0, b1, actions[int64 B x N+1]) backends/_kernel.pyx:275-279
 *
 * Each entry point below replaces one of those (see the per-function notes).
 * Differences are deliberate and B200-first: every call is batched over the
 * whole env range (no per-env host calls), all buffers are device pointers
 * borrowed from the caller (PyTorch allocates them; this library allocates only
 * its private read-only tables), and calls are asynchronous on a caller-given
 * CUDA stream.  Errors are returned as status codes with a thread-local
 * message from vy_last_error(); device-side range violations (an action index
 * outside [0, 2K]) set a sticky error word read by vy_poll_error().
 *
 * Plain C types only: no torch, no CUDA runtime types (streams are void*).
 */
#ifndef VOLTYARD_B200_H
#define VOLTYARD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VY_ABI_VERSION 1

/* status codes */
#define VY_OK 0
#define VY_ERR_ARG 1       /* bad argument (maps to ValueError)            */
#define VY_ERR_CUDA 2      /* CUDA runtime failure (maps to RuntimeError)  */
#define VY_ERR_UNSUPPORTED 3 /* configuration outside the compiled kernels */
#define VY_ERR_STATE 4     /* call order violated (maps to EpisodeDone)    */

/* action element types accepted by vy_step */
#define VY_ACT_U8 0
#define VY_ACT_I32 1
#define VY_ACT_I64 2

/* vy_step / vy_rollout flags */
#define VY_F_AUTO_RESET 1u   /* reset done envs to episode+1 inside the kernel (engine.py:460-462) */
#define VY_F_INFOS 2u        /* write the info block (engine.py:282-336 'StepOutputs')             */
#define VY_F_INJECT 4u       /* take arrival draws from vy_draws instead of the reference stream  */
#define VY_F_OUT_F64 8u      /* obs/reward buffers are float64 (exact drop-in) instead of float32  */

/*
 * Read-only model tables (host pointers; copied to the device by vy_create).
 * Field-for-field the content of the reference's KernelTables
 * (engine.py:30-104, built by build_tables engine.py:107-218).
 */
typedef struct vy_tables {
  /* station (topology.py:169-214) */
  int32_t n_ports, n_slots, n_nodes, max_passes;
  const double *volt, *imax_c, *imax_d, *eta_c, *eta_d, *i_denom; /* [n_ports] */
  const int32_t *kind, *order;                                     /* [n_ports] */
  const double *node_cap, *node_eta;                               /* [n_nodes] */
  const int32_t *node_ptr;                                         /* [n_nodes+1] */
  const int32_t *node_leaf;                                        /* [node_ptr[n_nodes]] */
  const int32_t *node_order;                                       /* [n_nodes] deepest first */
  /* station battery (engine.py:112-118, 149, 178) */
  int32_t battery_enabled;
  double b_volt, b_cap, b_rmax, b_tau, b_eta_c, b_eta_d, b_init_soc, b_imax, b_idenom;
  /* config (config.py:33-96) */
  int32_t k, episode_steps, steps_per_day, dt_min, horizon, obs_len, allow_discharge;
  double dt_h, p_sell, c_dt, beta;
  double alphas[8]; /* PENALTY_NAMES order (config.py:19-28) */
  /* exogenous data (data.py:40-183) */
  int32_t n_days, lam_len, has_moer, has_dgrid;
  double wk_scale, we_scale;
  const double *buy, *sellg;  /* [n_days*24] */
  const double *lam;          /* [lam_len] */
  const int8_t *weekday;      /* [n_days] */
  const double *moer, *dgrid; /* [n_days*24] (or [1] zeros when absent) */
  const double *sin_t, *cos_t;/* [steps_per_day] */
  /* car catalogue and user scenario */
  int32_t n_cat, stay_lo, stay_hi;
  const double *cat_cum, *cat_cap, *cat_rac, *cat_rdc, *cat_tau; /* [n_cat] */
  double soc_lo, soc_hi, frac_lo, frac_hi, p_charge;
} vy_tables;

/*
 * Device state, struct-of-arrays.  Per-port arrays are port-major [n_ports][ld]
 * (element (b, i) at i*ld + b) so a warp of 32 consecutive envs touches one
 * contiguous 256 B run per field and port.  Continuous quantities stay float64:
 * the kernels reproduce the reference's float64 arithmetic operation for
 * operation, which is what makes discrete state bit-exact at any batch size.
 * Replaces StateArrays (engine.py:221-279); cap/rbar/tau/rhat are not stored:
 * cap/rbar/tau come from the car-profile table via `meta`, rhat is recomputed
 * from soc exactly as the reference stores it (_kernel.pyx:389, 505).
 */
typedef struct vy_state {
  int64_t ld;            /* leading dimension (>= batch) of per-port arrays */
  double *port_i;        /* [n_ports][ld] i_drawn (A)                       */
  double *port_soc;      /* [n_ports][ld]                                   */
  double *port_de;       /* [n_ports][ld] remaining requested energy (kWh)  */
  int16_t *port_dtrem;   /* [n_ports][ld] remaining stay (steps)            */
  uint8_t *port_meta;    /* [n_ports][ld] bit0 occ, bit1 pref, bits2..7 profile */
  int32_t *step, *day, *episode; /* [B] */
  uint64_t *env_seed;    /* [B] */
  uint64_t *akey;        /* [B] arrival-stream prefix key of the current episode */
  double *b_i, *b_soc;   /* [B] station battery */
  double *ep_profit, *ep_reward, *ep_missing, *ep_energy; /* [B] */
  int32_t *ep_overtime, *ep_declined, *ep_departures;     /* [B] */
} vy_state;

/*
 * Per-step outputs.  obs is row-major [B][obs_len] (float32, or float64 with
 * VY_F_OUT_F64), reward [B] same dtype, done uint8 [B].  The info block is
 * written only with VY_F_INFOS and is feature-major [k][ld] (all NULL otherwise);
 * ep_stats and term_overtime are written whenever an episode ends.
 */
typedef struct vy_outputs {
  void *obs;
  void *reward;
  uint8_t *done;
  double *ep_stats;      /* [8][ld]  */
  int32_t *term_overtime;/* [ld]     */
  /* info block */
  double *breakdown;     /* [10][ld] */
  double *flows;         /* [5][ld]  */
  int32_t *declined, *arrivals_m, *dep_n; /* [ld] */
  int32_t *dep_port, *dep_overtime, *dep_early, *dep_pref; /* [n_ports][ld] */
  double *dep_missing, *dep_cap, *dep_soc;                 /* [n_ports][ld] */
  double *i_att, *i_used;  /* [n_slots][ld] */
  double *delivered;       /* [n_ports][ld] */
  double *b_delivered;     /* [ld] */
} vy_outputs;

/*
 * Injected arrival draws (VY_F_INJECT).  Env b samples
 * M_b = off[b+1] - off[b] cars this step; car j of env b is entry off[b]+j.
 * `profile` indexes the car-profile table (0..n_cat-1 are catalogue entries).
 * Replaces the draws of Stream(stream_key(seed, ep, 1, t)) consumed by
 * _kernel.pyx:461-488 (sample_arrival_count/sample_car/sample_user).
 */
typedef struct vy_draws {
  const int32_t *off;    /* [B+1] */
  const uint8_t *profile;
  const int32_t *stay;
  const double *soc0, *frac;
  const uint8_t *pref;
} vy_draws;

typedef struct vy_handle vy_handle;

int vy_abi_version(void);
const char *vy_last_error(void);

/* Build device tables for `batch` envs on `device`.  Replaces build_tables +
 * make_core (engine.py:370, 379-380; backends/__init__.py:43-47). */
int vy_create(const vy_tables *t, int64_t batch, int device, vy_handle **out);
int vy_destroy(vy_handle *h);

/* Register an extra car profile (capacity, AC/DC rate, tau) for state
 * injection (the reference's tests write cap/rbar/tau directly,
 * tests/helpers.py:163-189).  Returns the profile id (>= n_cat) or -1. */
int vy_add_profile(vy_handle *h, double cap, double r_ac, double r_dc, double tau);
/* Copy profile p's derived values to host: cap, r_ac, r_dc, tau. */
int vy_get_profile(vy_handle *h, int p, double out4[4]);

/* Borrow caller-owned device buffers (engine.py:375-378 ownership). */
int vy_bind(vy_handle *h, const vy_state *s, const vy_outputs *o);

/* Reset envs.  mask: device uint8 [B] (NULL = all).  episode_mode 0: episode
 * := 0 (first reset); 1: episode := episode+1 (engine.py:414-424).  The day
 * is drawn from Stream(stream_key(seed, episode, 0, 0)) (_kernel.pyx:239-261)
 * unless inj_day (device int32 [B]) is given.  Writes the reset observation. */
int vy_reset(vy_handle *h, const uint8_t *mask, int32_t episode_mode,
             const int32_t *inj_day, uint32_t flags, void *stream);

/* Reset the envs selected by `mask` (device uint8 [B], NULL = all) to the
 * explicit episode numbers `episodes` (device int32 [B]) — the per-env call
 * core.reset_env(b, episode) of the reference's plugin protocol
 * (_kernel.pyx:239-261; BatchEnv.reset / auto-reset, engine.py:414-424,
 * 459-462), batched into one launch.  Writes the reset observations. */
int vy_reset_episodes(vy_handle *h, const uint8_t *mask, const int32_t *episodes, uint32_t flags, void *stream);

/* Set the seed of every env: env_seed[b] = split_seed(master, b + index0)
 * (engine.py:371-372, 407-412).  Does not reset. */
int vy_seed_envs(vy_handle *h, int64_t master_seed, int64_t index0, void *stream);

/* One step of every env.  actions: device array of `dtype` with element
 * (b, slot) at b*row_stride + slot*col_stride.  Replaces step_range(0, B, a)
 * plus the auto-reset loop (engine.py:446-462). */
int vy_step(vy_handle *h, const void *actions, int32_t dtype, int64_t row_stride,
            int64_t col_stride, uint32_t flags, const vy_draws *inj, void *stream);

/* RandomPolicy.actions (policies.py:51-73) on device: row b uses the stream
 * stream_key(seed, b + index0, 2); `call` is the number of earlier calls.
 * Writes uint8 [B][n_ports+1]. */
int vy_random_actions(vy_handle *h, uint64_t seed, int64_t index0, int64_t call,
                      uint8_t *out, void *stream);

/* As vy_random_actions, with the call index read from (and then incremented
 * in) a device counter, so the launch can be replayed from a CUDA graph and
 * still draw the next call's actions every replay.  call_counter points to two
 * int64: the call index and a scratch word (0 between launches) the kernel's
 * blocks use to elect the one that advances the index. */
int vy_random_actions_dev(vy_handle *h, uint64_t seed, int64_t index0, int64_t *call_counter, uint8_t *out,
                          void *stream);

/* One step of every env with RandomPolicy actions generated inside the step
 * kernel: the fused form of the throughput_probe loop body
 * `env.step(policy.actions(obs))` (engine.py:541-545, policies.py:51-73).
 * The actions equal vy_random_actions(seed, index0, call) bit for bit; the
 * call index is `call`, plus *call_counter when call_counter is non-NULL (two
 * int64, as vy_random_actions_dev; the kernel advances word 0 by one, so a
 * graph replay draws the next call).  actions_out (NULL = not written)
 * receives the uint8 [B][n_ports+1] actions.  flags as vy_step (no
 * VY_F_INJECT). */
int vy_step_random(vy_handle *h, uint64_t seed, int64_t index0, int64_t call, int64_t *call_counter,
                   uint8_t *actions_out, uint32_t flags, void *stream);

/* Fused multi-step rollout: T steps with in-kernel RandomPolicy actions and
 * auto-reset, state held in registers across steps.  Step t writes obs to
 * obs + t*obs_step_stride (elements; 0 = overwrite one buffer), reward to
 * reward + t*rew_step_stride, done to done + t*rew_step_stride.  Equivalent to
 * T iterations of the throughput_probe loop (engine.py:541-545). */
int vy_rollout(vy_handle *h, int32_t T, uint64_t policy_seed, int64_t index0, int64_t call0,
               void *obs, int64_t obs_step_stride, void *reward, uint8_t *done,
               int64_t rew_step_stride, uint32_t flags, void *stream);

/* Sticky device error word (bit0: action index out of range).  Synchronises
 * the stream; clears the word when `clear` is non-zero. */
int vy_poll_error(vy_handle *h, int clear, void *stream, uint32_t *out);

/* Number of kernel launches issued through this handle (for bench accounting). */
int64_t vy_launch_count(vy_handle *h);

/* Diagnostics: which instantiation of the step kernel the last vy_step ran:
 * 1 / 2 = lean (obs/reward/done only, none of the optional model features,
 * staged uint8 actions; small / large capacity tree), 0 = generic, -1 = none
 * yet.  Results never depend on it (tests/test_gpu_parity.py runs both). */
int32_t vy_last_step_mode(vy_handle *h);

/* Launch shaping for batches that share the GPU with other handles (the
 * heterogeneous C5 batch runs one handle per station config on concurrent
 * streams): the persistent step kernel launches at most
 * ceil(tiles / (warps per CTA * k)) CTAs, so each warp steps about k 32-env
 * tiles.  Default 1 (as many CTAs as fit).  Results never depend on it. */
int vy_set_tiles_per_warp(vy_handle *h, int32_t k);
/* Small-batch kernel choice: 1 = one warp per env / one lane per port
 * (k_rollout_wide: low latency at small batches, e.g. config C1's 16 envs) for
 * vy_rollout and for vy_step with staged uint8 actions and auto-reset, 0 = one
 * thread per env, -1 = by batch size (default: vy_rollout goes wide at <= 4096
 * envs, vy_step stays on the tile kernel).  Wide needs a lean station without
 * a battery, <= 32 ports, float32 obs; otherwise the tile kernels run.
 * Outputs are identical. */
int vy_set_wide(vy_handle *h, int32_t mode);

/* PPO minibatch loss head in one pass (vy_ppo.cu): from bf16 head rows
 * (S slots x A logits, the value in padding column value_col, row stride ld)
 * and the stored actions, the per-sample {old log-prob, old value, advantage,
 * return} rows (float32 x 4, 16-byte aligned) and the advantage mean / std
 * (device, 2 floats): the log-probabilities, entropies, values, the clipped
 * surrogate + clipped value loss + entropy bonus of PAPER.md:465-490, and
 * their gradient with respect to the head rows (bf16, same layout) for the
 * mean loss.  stats (device, 4 floats, zeroed by the caller) receives the
 * sums of {loss, pg, vf, ent} over the N samples. */
int vy_ppo_loss(const void *logits, int64_t ld, const uint8_t *actions, int64_t N, int32_t S, int32_t A,
                const float *scal4, const float *adv_stats, float clip_eps, float vf_clip, float vf_coef,
                float ent_coef, int32_t value_col, void *grad, float *stats, void *stream);

/* x[i] *= *g for n bf16 values unless *g == 1 (device scalar; PPOLoss's
 * backward: the upstream gradient without a host sync). */
int vy_scale_bf16(void *x, int64_t n, const float *g, void *stream);

/* Heterogeneous batch in one launch (config C5).  The
 * reference steps one (config, station, dataset) per BatchEnv (engine.py:370,
 * SPEC.md:482); a multi handle stacks n bound group handles (each keeps its
 * own tables, state and outputs) and steps all of them with ONE persistent
 * kernel: global tile t -> group g by the per-tile config index tile0[],
 * the group's Params stacked in device memory, every distinct table set
 * staged once per CTA.  Actions are each group's device RandomPolicy rows
 * (policy_seeds[g], env index0[g]; policies.py:51-73), drawn in the kernel
 * as in vy_step_random; call_counter (device, may be NULL) as there.  Distinct
 * car-profile tables and station tables (<= 8 each) are staged once per CTA.  Every
 * group's outputs equal a vy_step_random of that group alone.  Create after
 * the group handles are bound (the Params snapshot their buffers). */
typedef struct vy_multi vy_multi;
int vy_multi_create(vy_handle *const *handles, int32_t n, const uint64_t *policy_seeds, const int64_t *index0,
                    vy_multi **out);
int vy_multi_step_random(vy_multi *m, int64_t call, int64_t *call_counter, void *stream);
/* out4 = {Spec mode, 16 * car-profile sets + station sets, warps per CTA, grid} */
int32_t vy_multi_info(vy_multi *m, int32_t *out4);
int64_t vy_multi_launch_count(vy_multi *m);
int vy_multi_destroy(vy_multi *m);

/* PPO support (config C3): generalised advantage estimation as a reverse
 * scan over a [T][B] rollout (float32 values/rewards, uint8 dones, last_value
 * [B]); writes advantages and returns [T][B].  Not part of the reference
 * (its trainer-free scope); the paper's PPO. */
int vy_gae(const float *values, const float *rewards, const uint8_t *dones, const float *last_value, int32_t T,
           int64_t B, float gamma, float lam, float *adv, float *ret, void *stream);

/* PPO head kernels (config C3), one warp per sample over logits rows of S
 * slots x A actions (dtype 0 = float32, 1 = bfloat16; row n starts at element
 * n*ld, ld >= S*A, so a GEMM output padded to an aligned width is read in
 * place):
 * vy_ppo_sample   Gumbel-max action per slot from `noise` ~ U[0,1) float32
 *                 [N][S][A] -> actions uint8 [N][S], log-probability float32 [N];
 * vy_ppo_head_fwd log-probability of `actions` and entropy, summed over slots;
 * vy_ppo_head_bwd gradient (logits' dtype and row stride, padding columns 0)
 *                 of g_lp*lp + g_ent*ent w.r.t. the logits (either upstream
 *                 gradient may be NULL = 0); with g_value non-NULL, padding
 *                 column value_col (S*A <= value_col < ld: a value head
 *                 sharing the GEMM) receives g_value[n] instead of 0. */
int vy_ppo_sample(const void *logits, int32_t dtype, int64_t ld, const float *noise, int64_t N, int32_t S, int32_t A,
                  uint8_t *actions, float *logp, void *stream);
/* vy_ppo_sample with the uniforms drawn in the kernel: element e of call c
 * uses splitmix64(mix(seed, c) + e*golden); counter = int64[2] on the device,
 * {c, scratch = 0}, c advanced by the launch itself (CUDA-graph friendly).
 * value (optional, float32 [N]) receives padding column value_col of each
 * row (S*A <= value_col < ld): a value head sharing the GEMM. */
int vy_ppo_sample_rng(const void *logits, int32_t dtype, int64_t ld, uint64_t seed, int64_t *counter, int64_t N,
                      int32_t S, int32_t A, uint8_t *actions, float *logp, float *value, int32_t value_col,
                      void *stream);
int vy_ppo_head_fwd(const void *logits, int32_t dtype, int64_t ld, const uint8_t *actions, int64_t N, int32_t S,
                    int32_t A, float *lp, float *ent, void *stream);
int vy_ppo_head_bwd(const void *logits, int32_t dtype, int64_t ld, const uint8_t *actions, int64_t N, int32_t S,
                    int32_t A, const float *g_lp, const float *g_ent, const float *g_value, int32_t value_col,
                    void *grad, void *stream);
/* PPO minibatch gather: dst row i = src row idx[i] for i < n, rows of
 * row_bytes bytes (a multiple of 16; src and dst 16-byte aligned). */
/* PPO rollout policy forward on the tensor cores (tcgen05.mma, TMEM
 * accumulators, bulk-async obs tiles): one launch per rollout step.
 * obs: float32 [N][obs_ld] (first obs_dim columns used); the actor-critic of
 * ppo.py (hidden 64: W1 [128 x obs_dim], Wa2/Wc2 [64 x 64], head [S*A x 64],
 * value [1 x 64]) pre-packed by the host in the UMMA K-major layout:
 * wpack bf16 blob of out[0] bytes, fpack out[1] floats (vy_policy_geometry
 * gives the sizes; ppo.pack_policy the layout).  Writes the sampled uint8
 * actions [N][S] (inverse-CDF categorical sampling, one uniform per (row,
 * slot) from the counter-based stream keyed by seed and counter[0], which the
 * kernel advances: counter = {call, scratch}), the log-probability [N] and
 * the value [N]; logits_out (NULL = not written) receives the bf16-rounded
 * logits [N][S*A] as float32.  Not part of the reference (trainer-free,
 * SPEC.md:14); the paper's PPO network. */
int vy_policy_geometry(int32_t obs_dim, int32_t obs_ld, int32_t S, int32_t A, int32_t out[4]);
int vy_policy_step(const float *obs, int64_t obs_ld, int64_t N, int32_t obs_dim, int32_t S, int32_t A,
                   const void *wpack, const float *fpack, uint64_t seed, int64_t *counter, uint8_t *actions,
                   float *logp, float *value, float *logits_out, void *stream);

/* The whole PPO rollout as ONE kernel launch (small batches: 16 envs per
 * CTA, one CTA per SM): T x {policy forward + sampling on the tensor cores
 * (the same arithmetic and sampling stream as vy_policy_step), env step (the
 * one-warp-per-env step, auto-reset)} and a last policy pass for the
 * bootstrap value.  Equivalent, bit for bit, to T + 1 vy_policy_step calls
 * interleaved with T vy_step calls on the sampled actions.  obs: float32
 * [T+1][B][obs_len] (row 0 = the current obs, read; rows 1..T written);
 * actions uint8 [T][B][S]; logp / reward float32 [T][B]; value float32
 * [T+1][B]; done uint8 [T][B]; S = n_ports + 1, A = 2k + 1; counter as for
 * vy_policy_step, advanced by T + 1.  VY_ERR_UNSUPPORTED unless the station
 * is lean without a battery and has <= 32 ports (callers then run the
 * per-step pair).  Not part of the reference (trainer-free). */
int vy_ppo_rollout(vy_handle *h, int32_t T, const void *wpack, const float *fpack, int32_t S, int32_t A,
                   uint64_t seed, int64_t *counter, float *obs, uint8_t *actions, float *logp, float *value,
                   float *reward, uint8_t *done, void *stream);

/* One PPO minibatch update for small batches in three launches (fp32):
 * vy_ppo_update_grad = forward of the ppo.py actor-critic from its live fp32
 * weights (weights[10]: the module's parameters in order — W1 [2H][K1], b1,
 * Wa2, ba2, Wh [NO][H], bh, Wc2, bc2, wv [1][H], bv; K1 = obs_dim rounded up
 * to 8, NO = S*A rounded up to 8, H = hidden = 64), the clipped PPO loss of
 * vy_ppo_loss with the advantages normalised over the minibatch, backward,
 * per-CTA partial gradients summed in CTA order into grad_out[P] (the flat
 * gradient, module order), the minibatch means {loss, pg, vf, ent} into
 * stats[4], *step += 1.  Rows: idx[M] into obs [*][obs_ld] float32, actions
 * [*][S] uint8, scal4 [*] float4 {old_lp, old_v, adv, ret}.
 * vy_ppo_update_adam = torch's clip_grad_norm_(max_grad_norm) coefficient
 * and Adam (betas, eps, lr read on the device, bias correction from *step)
 * on params[10] in place; exp_avg / exp_avg_sq [P] zero-initialised by the
 * caller.  A multi-GPU caller all-reduces grad_out between the two.
 * w1t: W1 transposed [K1][2H], which the first layer reads (coalesced); the
 * caller fills it from W1 and vy_ppo_update_adam keeps it in step.
 * adv_stats: {mean, std} of the minibatch's advantages, or NULL (computed by
 * every CTA); vy_ppo_adv_stats computes them for all minibatches of an
 * update at once (block e*nmb + k: rows perms[e][k*mb .. (k+1)*mb)).
 * vy_ppo_update_workspace: out = {P, work floats, grad CTAs, shared bytes}.
 * Not part of the reference (trainer-free). */
int vy_ppo_adv_stats(const float *scal4, const int64_t *perms, int64_t n, int32_t count, int32_t nmb, int64_t mb,
                     float *out, void *stream);
int vy_ppo_update_workspace(int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M, int64_t out[4]);
int vy_ppo_update_grad(const float *const *weights, const float *w1t, int32_t obs_dim, int32_t S, int32_t A, int32_t hidden,
                       const float *obs, int64_t obs_ld, const uint8_t *actions, const float *scal4,
                       const int64_t *idx, const float *adv_stats, int64_t M, float clip_eps, float vf_clip, float vf_coef, float ent_coef,
                       float *work, float *grad_out, float *stats, float *step, void *stream);
int vy_ppo_update_adam(float *const *params, float *w1t, int32_t obs_dim, int32_t S, int32_t A, int32_t hidden, int64_t M,
                       float *work, const float *grad, float *exp_avg, float *exp_avg_sq, const float *lr,
                       const float *step, float beta1, float beta2, float eps, float max_grad_norm, void *stream);

/* count pseudo-random permutations of 0..n-1 (n <= 2^30) into out
 * [count][n] int64 — the PPO update's minibatch shuffles, one launch per
 * update: element i maps through a keyed 4-round Feistel bijection on
 * [0, 4^h) >= n with cycle-walking (no sort), one key per permutation from
 * (seed, call, c).  counter = {call, scratch} on the device, advanced by one
 * per launch (graph replays draw fresh permutations). */
int vy_random_perms(int64_t n, int32_t count, uint64_t seed, int64_t *counter, int64_t *out, void *stream);

/* GAE (vy_gae's recurrence and roundings) written straight into the update's
 * per-sample rows: scal4 [T*B] float4 = {logp, value, advantage, return};
 * values / rewards / logp [T][B] float32, dones [T][B] uint8, last_value [B].
 * Small rollouts run as one block staging the inputs in shared memory. */
int vy_gae_scal(const float *values, const float *rewards, const uint8_t *dones, const float *last_value,
                const float *logp, int32_t T, int64_t B, float gamma, float lam, float *scal4, void *stream);

int vy_gather_rows(const void *src, int64_t row_bytes, const int64_t *idx, int64_t n, void *dst, void *stream);
/* Column sums (a linear layer's bias gradient): out[c] = sum over m < M of
 * g[m*ld + c], c < N; g float32 (dtype 0) or bfloat16 (1); out float32.
 * work: float32 scratch of VY_COLSUM_BANDS * N values.  Deterministic (no
 * atomics: per-band partial sums, then the bands added in order). */
#define VY_COLSUM_BANDS 2048
int vy_colsum(const void *g, int32_t dtype, int64_t M, int64_t N, int64_t ld, float *work, float *out,
              void *stream);

/* Diagnostics: compare the kernels' reciprocal-based division (div_rcp in
 * csrc/vy_device.cuh) with IEEE x / d on `samples_per_divisor` random
 * dividends for each divisor; *mismatches receives the count (0 = bit-exact). */
int vy_selftest_div(const double *divisors, int32_t nd, int64_t samples_per_divisor, uint64_t seed,
                    int64_t *mismatches);

#ifdef __cplusplus
}
#endif
#endif /* VOLTYARD_B200_H */
