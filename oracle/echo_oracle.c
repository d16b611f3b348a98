/*
 * echo_oracle.c -- plain, slow, obviously-correct CPU oracle for the Echo learner hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  The product path (paper_2508_05387_b200/) never
 * links, imports or calls it, and shares no code, header or constant with it.
 *
 * What it computes: one learner step of Echo's training swarm (arXiv 2508.05387, §2.4
 * :254-282, "consumes trajectory batches, applies a chosen RL algorithm ... step() interface
 * consuming mini-batches drawn from the shared buffer"), with the GRPO recipe of PAPER.md §3.1
 * :374-382, written out as its plain definition in fp64:
 *
 *   (1) version-lag filter + pack      PAPER.md :192 (param_version tag), :224 (strict
 *                                      t_train - t_infer > Delta_max), :201 ("lag one or more
 *                                      updates"); SPEC.md :344/:354 (min_version filter)
 *   (2) GRPO group-relative advantage  PAPER.md :374 (GRPO named); SPEC.md :206-214 formula
 *   (3) log pi(a|s) = z_a - logsumexp  PAPER.md :170-171 ("log pi_theta(a|s)" field)
 *   (4) clipped surrogate + KL         PAPER.md :278 ("PPO, KL-constrained PPO, GRPO");
 *                                      SPEC.md :219 (clipped ratio objective), :243 (eps = 0.2);
 *                                      KL coefficient PAPER.md :376-382
 *   (5) dL/dlogits                     PAPER.md :254-256 ("performs gradient updates")
 *
 * Readings of silent / ambiguous points (DESIGN.md "Readings" R1-R17 list them all):
 *   R1  keep a group iff t_train - v <= max_lag (drop iff strictly greater, PAPER.md :224)
 *   R3  version tags must be uniform inside a group; the drop is group-granular
 *   R4  survivors are compacted in ascending order, tokens rollout-major
 *   R5  KL term is the k3 estimator against pi_ref: exp(ref-logp) - (ref-logp) - 1
 *   R6  loss = sum_t l_t / N_global (token mean over all ranks' kept tokens)
 *   R7  population std, A = (r - mean)/(std + eps), eps = 1e-8 (SPEC.md :209, :213)
 *   R10 "clipped" uses strict inequalities; at equality the gradient flows
 *
 * Conventions: every float input is widened exactly to double; all arithmetic is IEEE double with
 * no FMA contraction (-ffp-contract=off); libm exp/log/sqrt.  The only fp32 rounding the oracle
 * performs is where the ABI fixes an fp32 output (the advantage table, R13).
 *
 * Parity pins (tests/test_oracle_*.py): brute-force pack over all 3^4 lag patterns; SPEC.md :212-214
 * worked advantage examples; logp = -ln V on uniform rows; spike closed form; old == new => rho = 1;
 * clip saturation => zero gradient row; central finite differences of the loss vs dlogits.
 * Nothing here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <float.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- status codes (the oracle's own copies; kept independent of include/echo.h) ---- */
enum { REF_OK = 0, REF_ERR_INVALID_ARGUMENT = 1 };
enum {
  REF_DATA_OK = 0,
  REF_DATA_FUTURE_VERSION = 1,   /* v > t_train: a rollout from a policy the learner never had */
  REF_DATA_MIXED_GROUP_VERSION = 2,
  REF_DATA_BAD_LENGTH = 3,       /* L not in [1, S] (SPEC.md :39, sequences have length >= 1) */
  REF_DATA_BAD_ACTION = 4,       /* action not in [0, V) */
  REF_DATA_CAPACITY = 5          /* packed tokens exceed the caller's capacity */
};

typedef struct {
  int32_t status;
  int32_t first_bad_rollout;
  int32_t n_groups_kept;
  int32_t n_rollouts_kept;
  int64_t n_tokens;
} echo_ref_pack_result;

static double widen_bf16(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double logit_at(const void* logits, int dtype, int64_t ld, int64_t row, int64_t v) {
  if (dtype == 0) return (double)((const float*)logits)[row * ld + v];
  return widen_bf16(((const uint16_t*)logits)[row * ld + v]);
}

/* ======================================================================================
 * (1) Version-lag filter + pack.
 *   PAPER.md :192  each rollout is annotated with a param_version tag.
 *   PAPER.md :224  the coordinator acts when t_train - t_infer > Delta_max (strict), bounding the
 *                  lag at Delta_max; a rollout with lag == max_lag is therefore still admissible.
 *   SPEC.md :344   pull returns trajectories with param_version >= min_version
 *                  (== t_train - max_lag here).
 *   SPEC.md :44-49 a RolloutBatch is prompt-major: prompt p owns rollouts [p*G, (p+1)*G).
 * Errors are reported as (rollout, check) lexicographic minimum: checks for rollout i in the
 * order FUTURE(1) < MIXED(2) < BAD_LENGTH(3) < BAD_ACTION(4); CAPACITY(5) only when nothing
 * else failed.  On any data error only status / first_bad_rollout are specified.
 * filter_mode (f3, SURVEY.md §8.6 "partial-group handling if per-rollout versions ever differ"):
 *   0 (group)   the group's versions must agree (MIXED otherwise); keep / drop whole groups (reading R3)
 *   1 (rollout) keep rollout i iff t_train - version[i] <= max_lag; groups may be partial, no MIXED check;
 *               n_groups_kept counts the groups with at least one kept rollout
 * ====================================================================================== */
int echo_ref_pack_batch(int32_t n_rollouts, int32_t group_size, int32_t max_len, int32_t vocab,
                        int64_t t_train, int32_t max_lag, int64_t rollout_base,
                        const int64_t* version, const int32_t* resp_len,
                        const int32_t* action, const float* old_logp, const float* ref_logp,
                        const float* aux, int64_t token_capacity,
                        int32_t* kept_rollout, int64_t* kept_offset,
                        int32_t* tok_slot, int32_t* tok_action, float* tok_old, float* tok_ref, float* tok_aux,
                        echo_ref_pack_result* result, int32_t filter_mode) {
  if (n_rollouts < 0 || group_size < 2 || max_len < 1 || vocab < 1 || max_lag < 0) return REF_ERR_INVALID_ARGUMENT;
  if (filter_mode != 0 && filter_mode != 1) return REF_ERR_INVALID_ARGUMENT;
  if (n_rollouts % group_size != 0) return REF_ERR_INVALID_ARGUMENT;
  const int64_t R = n_rollouts, G = group_size, S = max_len;

  int64_t best_key = INT64_MAX; /* key = rollout * 8 + check */
  int32_t n_groups_kept = 0, n_rollouts_kept = 0;
  int64_t n_tokens = 0;

  /* validation of every rollout, ascending */
  for (int64_t i = 0; i < R; ++i) {
    int64_t first = (i / G) * G;
    int64_t key = INT64_MAX;
    if (version[i] > t_train) key = i * 8 + REF_DATA_FUTURE_VERSION;
    else if (filter_mode == 0 && version[i] != version[first]) key = i * 8 + REF_DATA_MIXED_GROUP_VERSION;
    else if (resp_len[i] < 1 || resp_len[i] > max_len) key = i * 8 + REF_DATA_BAD_LENGTH;
    if (key < best_key) best_key = key;
  }

  /* filter: one decision per group from its (uniform) version, or one per rollout (filter_mode 1) */
  for (int64_t g = 0; g < R / G; ++g) {
    int any = 0;
    for (int64_t i = g * G; i < (g + 1) * G; ++i) {
      int64_t lag = t_train - (filter_mode == 0 ? version[g * G] : version[i]);
      if (lag > (int64_t)max_lag) continue;
      kept_rollout[n_rollouts_kept] = (int32_t)(rollout_base + i);
      kept_offset[n_rollouts_kept] = n_tokens;
      int64_t L = resp_len[i];
      if (L < 0) L = 0;
      if (L > S) L = S;
      n_tokens += L;
      n_rollouts_kept += 1;
      any = 1;
    }
    n_groups_kept += any;
  }
  kept_offset[n_rollouts_kept] = n_tokens;

  /* actions of kept rollouts, ascending rollout then position */
  for (int32_t k = 0; k < n_rollouts_kept; ++k) {
    int64_t i = (int64_t)kept_rollout[k] - rollout_base;
    int64_t L = kept_offset[k + 1] - kept_offset[k];
    for (int64_t j = 0; j < L; ++j) {
      int32_t a = action[i * S + j];
      if (a < 0 || a >= vocab) {
        int64_t key = i * 8 + REF_DATA_BAD_ACTION;
        if (key < best_key) best_key = key;
        break;
      }
    }
  }

  /* gather (only when it fits) */
  if (n_tokens <= token_capacity) {
    for (int32_t k = 0; k < n_rollouts_kept; ++k) {
      int64_t i = (int64_t)kept_rollout[k] - rollout_base;
      for (int64_t t = kept_offset[k]; t < kept_offset[k + 1]; ++t) {
        int64_t j = t - kept_offset[k];
        tok_slot[t] = k;
        tok_action[t] = action[i * S + j];
        tok_old[t] = old_logp[i * S + j];
        if (ref_logp && tok_ref) tok_ref[t] = ref_logp[i * S + j];
        if (aux && tok_aux) tok_aux[t] = aux[i * S + j];
      }
    }
  }

  result->n_groups_kept = n_groups_kept;
  result->n_rollouts_kept = n_rollouts_kept;
  result->n_tokens = n_tokens;
  if (best_key != INT64_MAX) {
    result->status = (int32_t)(best_key % 8);
    result->first_bad_rollout = (int32_t)(rollout_base + best_key / 8);
  } else if (n_tokens > token_capacity) {
    result->status = REF_DATA_CAPACITY;
    result->first_bad_rollout = -1;
  } else {
    result->status = REF_DATA_OK;
    result->first_bad_rollout = -1;
  }
  return REF_OK;
}

/* ======================================================================================
 * (2) GRPO group-relative advantage, SPEC.md :206-214 (the paper names GRPO at PAPER.md :374
 * without a formula; SPEC.md :243, :255 record the reconstruction):
 *     mean = (sum_i r_i) / G            (sequential fp64 sum, index order)
 *     std  = sqrt((sum_i (r_i - mean)^2) / G)   (population std, SPEC.md :213 worked example)
 *     A_i  = (r_i - mean) / (std + eps),  eps = 1e-8   -> rounded to fp32 (ABI output type)
 * adv_f64 (nullable) receives A before the fp32 rounding.
 * Stats: per group {sum A, sum A^2, sum r, sum r^2} (A as the fp32 value), then summed over groups
 * in ascending order; adv_stats = {sum A, sum A^2, sum r, sum r^2, n_zero_std_groups, n_rollouts}.
 * A group is the run of consecutive kept rollouts with the same kept_rollout[k] / G; with whole groups (pack
 * filter_mode 0) every run has G members, with per-rollout filtering (filter_mode 1) a run has its n_g <= G
 * surviving members and G is replaced by n_g in the mean and the std (f3 partial groups).
 * ====================================================================================== */
int echo_ref_group_advantage(int32_t n_rollouts_kept, int32_t group_size, float eps,
                             const float* reward, const int32_t* kept_rollout, int64_t rollout_base,
                             float* adv_slot, double* adv_f64, double* adv_stats) {
  if (group_size < 2 || n_rollouts_kept < 0) return REF_ERR_INVALID_ARGUMENT;
  const int64_t G = group_size;
  double tot[4] = {0, 0, 0, 0};
  double n_zero_std = 0;
  int64_t g1;
  for (int64_t g0 = 0; g0 < n_rollouts_kept; g0 = g1) {
    const int64_t grp = ((int64_t)kept_rollout[g0]) / G;
    g1 = g0 + 1;
    while (g1 < n_rollouts_kept && ((int64_t)kept_rollout[g1]) / G == grp) ++g1;
    const double n_g = (double)(g1 - g0);
    double sum = 0.0;
    for (int64_t k = g0; k < g1; ++k) sum = sum + (double)reward[kept_rollout[k] - rollout_base];
    double mean = sum / n_g;
    double ss = 0.0;
    for (int64_t k = g0; k < g1; ++k) {
      double d = (double)reward[kept_rollout[k] - rollout_base] - mean;
      ss = ss + d * d;
    }
    double std = sqrt(ss / n_g);
    if (std == 0.0) n_zero_std += 1.0;
    double part[4] = {0, 0, 0, 0};
    for (int64_t k = g0; k < g1; ++k) {
      double r = (double)reward[kept_rollout[k] - rollout_base];
      double a64 = (r - mean) / (std + (double)eps);
      float a = (float)a64;
      adv_slot[k] = a;
      if (adv_f64) adv_f64[k] = a64;
      part[0] = part[0] + (double)a;
      part[1] = part[1] + (double)a * (double)a;
      part[2] = part[2] + r;
      part[3] = part[3] + r * r;
    }
    for (int q = 0; q < 4; ++q) tot[q] = tot[q] + part[q];
  }
  adv_stats[0] = tot[0];
  adv_stats[1] = tot[1];
  adv_stats[2] = tot[2];
  adv_stats[3] = tot[3];
  adv_stats[4] = n_zero_std;
  adv_stats[5] = (double)n_rollouts_kept;
  return REF_OK;
}

/* ======================================================================================
 * (3)-(5) per packed token t (one row of the [tokens x vocab] logits):
 *   (3) m = max_v z_v;  lse = m + log sum_v exp(z_v - m);  logp = z_a - lse      PAPER.md :170
 *   (4) rho  = exp(logp - old)                                                    SPEC.md :219
 *       clipped = (A > 0 and rho > 1+eps_hi) or (A < 0 and rho < 1-eps_lo)        (R10)
 *       pg   = max(-A rho, -A clip(rho, 1-eps_lo, 1+eps_hi))                      SPEC.md :219
 *       kl   = exp(ref - logp) - (ref - logp) - 1     (only when beta > 0)        (R5)
 *       l_t  = pg + beta kl;   L = sum_t l_t / N_global                           (R6)
 *   (5) dl/dlogp = [not clipped](-A rho) + beta (1 - exp(ref - logp))
 *       c_t = grad_scale * dl/dlogp / N_global
 *       d[t,v] = c_t (delta_{v,a} - exp(z_v - lse))                               PAPER.md :254
 * flags: bit0 = clipped; bit1 = non-finite (lse, logp, rho, l_t or c_t not a finite value that an
 * fp32 output can hold -- R11).
 * stats (nullable, sequential fp64 over rows): {sum l, sum (logp-old), sum kl_k3 (if ref),
 *   n_clipped, n_nonfinite, rho_min, rho_max, sum logp, n_rows, sum rho, sum w l}, rho stats over
 *   finite rows only.
 * f4 options: tok_adv / tok_weight (nullable, see adv_of), clip_dual (c > 1: for A < 0 the loss is capped at
 *   -A c with zero gradient), kl_estimator (REF_KL_*), and the entropy bonus (entropy_coef eta >= 0):
 *       H_t  = -sum_v p_v log p_v   (p_v = exp(z_v - lse); masked -inf logits contribute 0, the limit p log p -> 0)
 *       l_t  = pg + beta kl - eta H_t
 *       dH/dz_v = -p_v (log p_v + H_t), so  d[t,v] = c_t (delta_{v,a} - p_v) + s w_t eta p_v (log p_v + H_t)
 *   tok_entropy (nullable) receives H_t; with eta > 0, H_t joins the non-finite check.
 * dlogits (nullable) is [n_rows x vocab] doubles.
 * ====================================================================================== */
static int fits_f32(double x) { return isfinite(x) && fabs(x) <= (double)FLT_MAX; }

/* The KL estimators of f4 (x = ref - logp): k3 = e^x - x - 1 (default, R5), k1 = logp - ref, k2 = (logp - ref)^2/2;
 * kl_value / kl_dlogp return the estimator and its derivative with respect to logp. */
enum { REF_KL_K3 = 0, REF_KL_K1 = 1, REF_KL_K2 = 2 };
static double kl_value(int est, double x) {
  if (est == REF_KL_K1) return -x;
  if (est == REF_KL_K2) return 0.5 * x * x;
  return exp(x) - x - 1.0;
}
static double kl_dlogp(int est, double x) {
  if (est == REF_KL_K1) return 1.0;
  if (est == REF_KL_K2) return -x;
  return 1.0 - exp(x);
}

/* Per-token advantage (f4: tok_adv, e.g. PPO-GAE, else the rollout's GRPO advantage) and loss weight
 * (f4: tok_weight, e.g. sequence-mean aggregation, else 1 / N_global -- reading R6). */
static double adv_of(const float* tok_adv, const int32_t* tok_slot, const float* adv_slot, int64_t t) {
  return tok_adv ? (double)tok_adv[t] : (double)adv_slot[tok_slot[t]];
}

int echo_ref_policy_loss(int64_t n_rows, int32_t vocab, int64_t ld, int32_t dtype, const void* logits,
                         const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                         const int32_t* tok_slot, const float* adv_slot, const float* tok_adv,
                         const float* tok_weight, double n_global,
                         float clip_low, float clip_high, float clip_dual, float kl_coef, int32_t kl_estimator,
                         float grad_scale, float entropy_coef,
                         double* tok_logp, double* tok_loss, uint8_t* tok_flags, double* tok_coef,
                         double* tok_entropy, double* dlogits, double* stats) {
  if (n_rows < 0 || vocab < 1 || ld < vocab || (dtype != 0 && dtype != 1)) return REF_ERR_INVALID_ARGUMENT;
  if (kl_coef > 0.0f && tok_ref == NULL) return REF_ERR_INVALID_ARGUMENT;
  if (kl_estimator < REF_KL_K3 || kl_estimator > REF_KL_K2) return REF_ERR_INVALID_ARGUMENT;
  const double lo = 1.0 - (double)clip_low, hi = 1.0 + (double)clip_high;
  const double beta = (double)kl_coef, dual = (double)clip_dual, eta = (double)entropy_coef;
  if (entropy_coef < 0.0f) return REF_ERR_INVALID_ARGUMENT;

#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < n_rows; ++t) {
    /* (3) log-softmax at the sampled action */
    double m = -INFINITY;
    int has_nan = 0;
    for (int64_t v = 0; v < vocab; ++v) {
      double z = logit_at(logits, dtype, ld, t, v);
      if (isnan(z)) has_nan = 1;
      if (z > m) m = z;
    }
    double s = 0.0;
    for (int64_t v = 0; v < vocab; ++v) s = s + exp(logit_at(logits, dtype, ld, t, v) - m);
    double lse = (has_nan || !isfinite(m)) ? NAN : m + log(s);
    int32_t a = tok_action[t];
    double logp = logit_at(logits, dtype, ld, t, a) - lse;

    /* (4) clipped importance-ratio surrogate + optional KL to the reference policy */
    double A = adv_of(tok_adv, tok_slot, adv_slot, t);
    double rho = exp(logp - (double)tok_old[t]);
    int clipped = (A > 0.0 && rho > hi) || (A < 0.0 && rho < lo);
    double rho_c = rho < lo ? lo : (rho > hi ? hi : rho);
    double un = -A * rho, cl = -A * rho_c;
    double pg = un > cl ? un : cl;
    if (dual > 1.0 && A < 0.0 && pg > -A * dual) { /* dual clip: loss capped at -A c, no gradient */
      pg = -A * dual;
      clipped = 1;
    }
    double kl = 0.0, dkl = 0.0;
    if (beta > 0.0) {
      double x = (double)tok_ref[t] - logp;
      kl = kl_value(kl_estimator, x);
      dkl = kl_dlogp(kl_estimator, x);
    }
    /* f4 entropy bonus: H = -sum_v p_v log p_v over the unmasked logits */
    double H = 0.0;
    if (eta > 0.0 || tok_entropy) {
      for (int64_t v = 0; v < vocab; ++v) {
        double z = logit_at(logits, dtype, ld, t, v);
        if (z == -INFINITY) continue;
        double lp = z - lse;
        H = H - exp(lp) * lp;
      }
    }
    double loss = pg + beta * kl - eta * H;
    double dl_dlogp = (clipped ? 0.0 : -A * rho) + beta * dkl;
    double w = tok_weight ? (double)tok_weight[t] : 1.0 / n_global;
    double c = (double)grad_scale * w * dl_dlogp;
    double e = (double)grad_scale * w * eta;
    int nonfinite = !(fits_f32(lse) && fits_f32(logp) && fits_f32(rho) && fits_f32(loss) && fits_f32(c) &&
                      (eta == 0.0 || fits_f32(H)));

    tok_logp[t] = logp;
    tok_loss[t] = loss;
    tok_flags[t] = (uint8_t)((clipped ? 1 : 0) | (nonfinite ? 2 : 0));
    if (tok_coef) tok_coef[t] = c;
    if (tok_entropy) tok_entropy[t] = H;

    /* (5) gradient of the loss with respect to every logit of the row */
    if (dlogits) {
      for (int64_t v = 0; v < vocab; ++v) {
        double z = logit_at(logits, dtype, ld, t, v);
        double p = exp(z - lse);
        double g = c * ((v == a ? 1.0 : 0.0) - p);
        if (eta > 0.0 && z != -INFINITY) g = g + e * p * ((z - lse) + H);
        dlogits[t * (int64_t)vocab + v] = g;
      }
    }
  }

  if (stats) {
    double acc[11] = {0, 0, 0, 0, 0, INFINITY, -INFINITY, 0, 0, 0, 0};
    for (int64_t t = 0; t < n_rows; ++t) {
      double logp = tok_logp[t];
      acc[0] = acc[0] + tok_loss[t];
      acc[1] = acc[1] + (logp - (double)tok_old[t]);
      if (tok_ref) {
        double x = (double)tok_ref[t] - logp;
        acc[2] = acc[2] + (exp(x) - x - 1.0);
      }
      acc[3] = acc[3] + (double)(tok_flags[t] & 1);
      acc[4] = acc[4] + (double)((tok_flags[t] >> 1) & 1);
      if (!(tok_flags[t] & 2)) {
        double rho = exp(logp - (double)tok_old[t]);
        if (rho < acc[5]) acc[5] = rho;
        if (rho > acc[6]) acc[6] = rho;
        acc[9] = acc[9] + rho;
      }
      acc[7] = acc[7] + logp;
      acc[8] = acc[8] + 1.0;
      acc[10] = acc[10] + (tok_weight ? (double)tok_weight[t] : 1.0) * tok_loss[t];
    }
    for (int q = 0; q < 11; ++q) stats[q] = acc[q];
  }
  return REF_OK;
}

/* ======================================================================================
 * f4: PPO-GAE advantages (Schulman et al., generalised advantage estimation) over each
 * trajectory's per-step rewards and values (PAPER.md :163-164, :170-171), written as its definition:
 *   delta_t = r_t + gamma V_{t+1} - V_t  (V_L = bootstrap or 0),  A_t = delta_t + gamma lambda A_{t+1} (A_L = 0),
 *   returns_t = A_t + V_t;  fp64, backwards over t, rounded to fp32.
 * ====================================================================================== */
int echo_ref_gae_advantage(int32_t n_rollouts, int32_t max_len, const int32_t* resp_len, const float* rewards,
                           const float* values, const float* bootstrap, float gamma, float lam, float* adv,
                           float* returns) {
  if (n_rollouts < 0 || max_len < 1) return REF_ERR_INVALID_ARGUMENT;
  const double g = (double)gamma, gl = (double)gamma * (double)lam;
  for (int64_t i = 0; i < n_rollouts; ++i) {
    int64_t L = resp_len[i] < 0 ? 0 : (resp_len[i] > max_len ? max_len : resp_len[i]);
    double v_next = bootstrap ? (double)bootstrap[i] : 0.0;
    double a = 0.0;
    for (int64_t t = L - 1; t >= 0; --t) {
      double v = (double)values[i * max_len + t];
      double delta = ((double)rewards[i * max_len + t] + g * v_next) - v;
      a = delta + gl * a;
      adv[i * max_len + t] = (float)a;
      if (returns) returns[i * max_len + t] = (float)(a + v);
      v_next = v;
    }
  }
  return REF_OK;
}

/* ======================================================================================
 * f1: forward-only token log-probs, the log pi_theta(a|s) field of PAPER.md :170 that a
 * trainer recomputes for old_logp (PAPER.md :162) and ref_logp (KL reference, PAPER.md :278):
 *   lse_t = m + log sum_v exp(z_v - m),  m = max_v z_v;   logp_t = z[t, a_t] - lse_t
 * flags bit1 = non-finite (lse or logp not a finite fp32 value), as in echo_ref_policy_loss.
 * ====================================================================================== */
int echo_ref_token_logp(int64_t n_rows, int32_t vocab, int64_t ld, int32_t dtype, const void* logits,
                        const int32_t* tok_action, double* tok_logp, double* tok_lse, uint8_t* tok_flags) {
  if (n_rows < 0 || vocab < 1 || ld < vocab || (dtype != 0 && dtype != 1)) return REF_ERR_INVALID_ARGUMENT;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < n_rows; ++t) {
    double m = -INFINITY;
    int has_nan = 0;
    for (int64_t v = 0; v < vocab; ++v) {
      double z = logit_at(logits, dtype, ld, t, v);
      if (isnan(z)) has_nan = 1;
      if (z > m) m = z;
    }
    double s = 0.0;
    for (int64_t v = 0; v < vocab; ++v) s = s + exp(logit_at(logits, dtype, ld, t, v) - m);
    double lse = (has_nan || !isfinite(m)) ? NAN : m + log(s);
    double logp = logit_at(logits, dtype, ld, t, tok_action[t]) - lse;
    tok_logp[t] = logp;
    if (tok_lse) tok_lse[t] = lse;
    if (tok_flags) tok_flags[t] = (uint8_t)((fits_f32(lse) && fits_f32(logp)) ? 0 : 2);
  }
  return REF_OK;
}

/* Scalar loss of a set of rows as a function of the logits, for finite-difference pins of (5):
 * returns grad_scale * sum_t w_t l_t (w_t = tok_weight[t] or 1 / N_global), i.e. the quantity whose gradient
 * dlogits is. */
double echo_ref_scaled_loss(int64_t n_rows, int32_t vocab, int64_t ld, const double* logits,
                            const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                            const int32_t* tok_slot, const float* adv_slot, const float* tok_adv,
                            const float* tok_weight, double n_global, float clip_low, float clip_high,
                            float clip_dual, float kl_coef, int32_t kl_estimator, float grad_scale,
                            float entropy_coef) {
  const double lo = 1.0 - (double)clip_low, hi = 1.0 + (double)clip_high;
  const double beta = (double)kl_coef, dual = (double)clip_dual, eta = (double)entropy_coef;
  double total = 0.0;
  for (int64_t t = 0; t < n_rows; ++t) {
    const double* z = logits + t * ld;
    double m = -INFINITY;
    for (int64_t v = 0; v < vocab; ++v) if (z[v] > m) m = z[v];
    double s = 0.0;
    for (int64_t v = 0; v < vocab; ++v) s = s + exp(z[v] - m);
    double lse = m + log(s);
    double logp = z[tok_action[t]] - lse;
    double H = 0.0;
    for (int64_t v = 0; v < vocab; ++v)
      if (z[v] != -INFINITY) H = H - exp(z[v] - lse) * (z[v] - lse);
    double A = adv_of(tok_adv, tok_slot, adv_slot, t);
    double rho = exp(logp - (double)tok_old[t]);
    double rho_c = rho < lo ? lo : (rho > hi ? hi : rho);
    double un = -A * rho, cl = -A * rho_c;
    double pg = un > cl ? un : cl;
    if (dual > 1.0 && A < 0.0 && pg > -A * dual) pg = -A * dual;
    double kl = 0.0;
    if (beta > 0.0) kl = kl_value(kl_estimator, (double)tok_ref[t] - logp);
    double w = tok_weight ? (double)tok_weight[t] : 1.0 / n_global;
    total = total + w * (pg + beta * kl - eta * H);
  }
  return (double)grad_scale * total;
}

/* ======================================================================================
 * f3: the CSR of (1) rebuilt from kept-rollout lengths after token-balanced resharding
 * (PAPER.md :224 drops whole groups; rollouts are then moved between ranks whole):
 *   kept_offset[0] = 0, kept_offset[i+1] = kept_offset[i] + max(lengths[i], 0);  tok_slot[t] = i for
 *   kept_offset[i] <= t < kept_offset[i+1].
 * ====================================================================================== */
int echo_ref_csr_from_lengths(int32_t n, const int32_t* lengths, int64_t* kept_offset, int32_t* tok_slot) {
  if (n < 0) return REF_ERR_INVALID_ARGUMENT;
  kept_offset[0] = 0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t len = lengths[i] > 0 ? lengths[i] : 0;
    kept_offset[i + 1] = kept_offset[i] + len;
    if (tok_slot)
      for (int64_t t = kept_offset[i]; t < kept_offset[i + 1]; ++t) tok_slot[t] = i;
  }
  return REF_OK;
}

/* ======================================================================================
 * f2: the LM head fused with the log-softmax-and-gather of (3), forward only.  The logits are
 * the LM head's output z[t, v] = sum_k h[t, k] W[v, k] (the model's final projection, PAPER.md :254-261
 * "the learner ... computes gradients"), so the fused form never materialises the [tokens x vocab] matrix:
 *   z[t, v] = sum_k h[t, k] W[v, k]   (bf16 inputs widened exactly to fp64, fp64 sums in k order)
 *   lse_t = m + log sum_v exp(z[t, v] - m),  m = max_v z[t, v];   logp_t = z[t, a_t] - lse_t
 * hidden: bf16 bit patterns [n_rows x d] row-major; weight: bf16 [vocab x d] row-major.
 * tok_entropy (nullable): H_t = -sum_v p_v log p_v, p_v = exp(z[t, v] - lse_t) (the f4 entropy of the policy).
 * ====================================================================================== */
int echo_ref_lmhead_logp(int64_t n_rows, int32_t d, int32_t vocab, const uint16_t* hidden, const uint16_t* weight,
                         const int32_t* tok_action, double* tok_logp, double* tok_lse, double* tok_entropy) {
  if (n_rows < 0 || d < 1 || vocab < 1) return REF_ERR_INVALID_ARGUMENT;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_rows; ++t) {
    double* z = (double*)malloc(sizeof(double) * (size_t)vocab);
    double m = -INFINITY;
    for (int64_t v = 0; v < vocab; ++v) {
      double acc = 0.0;
      for (int64_t k = 0; k < d; ++k)
        acc = acc + widen_bf16(hidden[t * d + k]) * widen_bf16(weight[v * d + k]);
      z[v] = acc;
      if (acc > m) m = acc;
    }
    double s = 0.0;
    for (int64_t v = 0; v < vocab; ++v) s = s + exp(z[v] - m);
    double lse = m + log(s);
    tok_logp[t] = z[tok_action[t]] - lse;
    if (tok_lse) tok_lse[t] = lse;
    if (tok_entropy) {
      double H = 0.0;
      for (int64_t v = 0; v < vocab; ++v) H = H - exp(z[v] - lse) * (z[v] - lse);
      tok_entropy[t] = H;
    }
    free(z);
  }
  return REF_OK;
}

/* ======================================================================================
 * f3: the staleness histogram of a step -- the per-step log record of SPEC.md :604
 * ({step, version, mean_return, staleness_histogram}) and the buffer's version_histogram (SPEC.md :373), with
 * staleness = t_train - param_version (SPEC.md :701; PAPER.md :192, :224).  Per rollout i of group g = i / G:
 *   lag_i = t_train - version[i];  kept_i = (t_train - version[g G] <= max_lag)   (the filter of (1), reading R1/R3;
 *   filter_mode 1: t_train - version[i] <= max_lag, the per-rollout filter)
 *   bin(lag) = 0 if lag < 0 (a future version), 1 + lag if 0 <= lag < n_bins, n_bins + 1 otherwise
 *   hist[0][bin] += kept_i, hist[1][bin] += !kept_i,
 *   hist[2][bin] += kept_i * L_i, hist[3][bin] += !kept_i * L_i,   L_i = min(max(resp_len[i], 0), max_len)
 * hist: int64 [4][n_bins + 2].
 * ====================================================================================== */
int echo_ref_staleness_histogram(int32_t n_rollouts, int32_t group_size, int32_t max_len, int64_t t_train,
                                 int32_t max_lag, const int64_t* version, const int32_t* resp_len, int32_t n_bins,
                                 int64_t* hist, int32_t filter_mode) {
  if (n_rollouts < 0 || group_size < 1 || n_rollouts % group_size != 0 || max_len < 1 || n_bins < 1)
    return REF_ERR_INVALID_ARGUMENT;
  const int32_t nb = n_bins + 2;
  for (int32_t k = 0; k < 4 * nb; ++k) hist[k] = 0;
  for (int32_t i = 0; i < n_rollouts; ++i) {
    int64_t lag = t_train - version[i];
    int64_t lag0 = t_train - version[filter_mode == 0 ? (i / group_size) * group_size : i];
    int kept = lag0 <= (int64_t)max_lag;
    int32_t bin = lag < 0 ? 0 : (lag < n_bins ? (int32_t)lag + 1 : n_bins + 1);
    int64_t L = resp_len[i] < 0 ? 0 : (resp_len[i] > max_len ? max_len : resp_len[i]);
    hist[(kept ? 0 : 1) * nb + bin] += 1;
    hist[(kept ? 2 : 3) * nb + bin] += L;
  }
  return REF_OK;
}

/* ======================================================================================
 * (4) from log-probs alone (with f1 / f2, which produce logp without the logits): the per-token surrogate, KL,
 * entropy bonus and gradient coefficient of echo_ref_policy_loss, restated from logp (and the row entropy H when
 * entropy_coef > 0):
 *   rho = exp(logp - old); pg = max(-A rho, -A clip(rho, 1-lo, 1+hi)); dual clip; kl by estimator;
 *   l_t = pg + beta kl - eta H;  c_t = grad_scale w_t ([not clipped](-A rho) + beta dkl/dlogp)
 * flags: bit0 clipped, bit1 non-finite (logp, rho, l_t, c_t not representable in fp32).
 * ====================================================================================== */
int echo_ref_loss_from_logp(int64_t n, const double* tok_logp, const double* tok_entropy, const float* tok_old,
                            const float* tok_ref, const int32_t* tok_slot, const float* adv_slot, const float* tok_adv,
                            const float* tok_weight, double n_global, float clip_low, float clip_high, float clip_dual,
                            float kl_coef, int32_t kl_estimator, float grad_scale, float entropy_coef,
                            double* tok_loss, uint8_t* tok_flags, double* tok_coef) {
  if (n < 0 || (kl_coef > 0.0f && !tok_ref) || (entropy_coef > 0.0f && !tok_entropy)) return REF_ERR_INVALID_ARGUMENT;
  const double lo = 1.0 - (double)clip_low, hi = 1.0 + (double)clip_high;
  const double beta = (double)kl_coef, dual = (double)clip_dual, eta = (double)entropy_coef;
  for (int64_t t = 0; t < n; ++t) {
    double logp = tok_logp[t];
    double A = adv_of(tok_adv, tok_slot, adv_slot, t);
    double rho = exp(logp - (double)tok_old[t]);
    int clipped = (A > 0.0 && rho > hi) || (A < 0.0 && rho < lo);
    double rho_c = rho < lo ? lo : (rho > hi ? hi : rho);
    double un = -A * rho, cl = -A * rho_c;
    double pg = un > cl ? un : cl;
    if (dual > 1.0 && A < 0.0 && pg > -A * dual) {
      pg = -A * dual;
      clipped = 1;
    }
    double kl = 0.0, dkl = 0.0;
    if (beta > 0.0) {
      double x = (double)tok_ref[t] - logp;
      kl = kl_value(kl_estimator, x);
      dkl = kl_dlogp(kl_estimator, x);
    }
    double H = eta > 0.0 ? tok_entropy[t] : 0.0;
    double loss = pg + beta * kl - eta * H;
    double w = tok_weight ? (double)tok_weight[t] : 1.0 / n_global;
    double c = (double)grad_scale * w * ((clipped ? 0.0 : -A * rho) + beta * dkl);
    int nonfinite = !(fits_f32(logp) && fits_f32(rho) && fits_f32(loss) && fits_f32(c));
    tok_loss[t] = loss;
    tok_flags[t] = (uint8_t)((clipped ? 1 : 0) | (nonfinite ? 2 : 0));
    if (tok_coef) tok_coef[t] = c;
  }
  return REF_OK;
}

/* ======================================================================================
 * f2 backward ("backward recomputes to give dhidden and dW"): the gradient of the step objective
 * J = sum_t c-weighted l_t through the LM head z = h W^T (PAPER.md :254-261, the learner "performs gradient updates"
 * on the policy; the logits gradient is (5), PAPER.md :254-256):
 *   z[t, v] = sum_k h[t, k] W[v, k];  lse_t, p[t, v] = exp(z[t, v] - lse_t), H_t = -sum_v p log p   (as lmhead_logp)
 *   D[t, v] = c_t (delta_{v, a_t} - p[t, v]) + e_t p[t, v] (log p[t, v] + H_t)      (the (5) row of echo_ref_policy_loss)
 *   dhidden[t, k] = sum_v D[t, v] W[v, k]      dweight[v, k] = sum_t D[t, v] h[t, k]
 * c_t = the token's gradient coefficient (echo_ref_loss_from_logp's tok_coef), e_t = grad_scale w_t eta (nullable:
 * 0).  hidden / weight are fp64 (the bf16 inputs widened exactly by the caller).  dlogits [n x V], dhidden [n x d],
 * dweight [V x d]: each nullable.  All sums in index order, fp64.
 * ====================================================================================== */
int echo_ref_lmhead_backward(int64_t n_rows, int32_t d, int32_t vocab, const double* hidden, const double* weight,
                             const int32_t* tok_action, const double* tok_coef, const double* tok_ecoef,
                             double* dlogits, double* dhidden, double* dweight) {
  if (n_rows < 0 || d < 1 || vocab < 1) return REF_ERR_INVALID_ARGUMENT;
  double* D = (double*)malloc(sizeof(double) * (size_t)(n_rows > 0 ? n_rows : 1) * (size_t)vocab);
  if (!D) return REF_ERR_INVALID_ARGUMENT;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_rows; ++t) {
    double* z = D + t * vocab;
    double m = -INFINITY;
    for (int64_t v = 0; v < vocab; ++v) {
      double acc = 0.0;
      for (int64_t k = 0; k < d; ++k) acc = acc + hidden[t * d + k] * weight[v * d + k];
      z[v] = acc;
      if (acc > m) m = acc;
    }
    double s = 0.0;
    for (int64_t v = 0; v < vocab; ++v) s = s + exp(z[v] - m);
    double lse = m + log(s);
    double H = 0.0;
    for (int64_t v = 0; v < vocab; ++v) H = H - exp(z[v] - lse) * (z[v] - lse);
    double c = tok_coef[t], e = tok_ecoef ? tok_ecoef[t] : 0.0;
    for (int64_t v = 0; v < vocab; ++v) {
      double lp = z[v] - lse, p = exp(lp);
      double delta = (v == tok_action[t]) ? 1.0 : 0.0;
      z[v] = c * (delta - p) + e * p * (lp + H); /* D[t, v] overwrites z[t, v] */
    }
  }
  if (dlogits)
    for (int64_t i = 0; i < n_rows * (int64_t)vocab; ++i) dlogits[i] = D[i];
  if (dhidden) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_rows; ++t)
      for (int64_t k = 0; k < d; ++k) {
        double acc = 0.0;
        for (int64_t v = 0; v < vocab; ++v) acc = acc + D[t * vocab + v] * weight[v * d + k];
        dhidden[t * d + k] = acc;
      }
  }
  if (dweight) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < vocab; ++v)
      for (int64_t k = 0; k < d; ++k) {
        double acc = 0.0;
        for (int64_t t = 0; t < n_rows; ++t) acc = acc + D[t * vocab + v] * hidden[t * d + k];
        dweight[v * d + k] = acc;
      }
  }
  free(D);
  return REF_OK;
}

/* Thread count of the OpenMP loops above (timing the oracle on one core vs all cores; no effect on results). */
void echo_ref_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
