/*
 * echo.h -- C ABI of the B200-native learner hot path of Echo (arXiv 2508.05387).
 *
 * One learner step of the training swarm (§2.4 :254-282: the trainer's step() "consuming
 * mini-batches drawn from the shared buffer") over version-tagged rollouts (PAPER.md :192) runs:
 *
 *   echo_pack_batch           (1) version-lag filter + pack        PAPER.md :192, :201, :224
 *   echo_group_advantage      (2) GRPO group-relative advantage    PAPER.md :374; SPEC.md :206-214
 *   echo_policy_loss_fwd_bwd  (3) log-softmax gather  (4) clipped surrogate + KL  (5) dL/dlogits in place
 *                                                                  PAPER.md :170-171, :278, :376-382
 *   echo_loss_stats           fixed-order fp64 reduction of the per-token outputs (statistics)
 *
 * SURVEY.md §8.6 NEXT rows:
 *   echo_token_logp                   f1  forward-only log-probs (read-only pass)
 *   echo_lmhead_logp                  f2  LM head fused with the log-prob on the tcgen05 tensor cores
 *   echo_loss_from_logp, echo_lmhead_dlogits, echo_lmhead_backward, echo_lmhead_logits,
 *   echo_lmhead_policy_loss_fwd_bwd
 *                                     f2  training step through the LM head: (4) from logp, D recomputed on the
 *                                         tensor cores, dhidden / dweight
 *   echo_pack_batch_v2, echo_staleness_histogram, echo_csr_from_lengths
 *                                     f3  per-rollout staleness filter, staleness histogram, CSR after resharding
 *   echo_policy_loss_fwd_bwd_v2, echo_gae_advantage
 *                                     f4  loss variants (per-token advantages / weights, k1/k2/k3, dual clip,
 *                                         entropy bonus) and PPO-GAE
 *
 * Conventions shared by every entry point
 *   - All array pointers are DEVICE pointers owned by the caller (e.g. torch allocations).  The library
 *     never allocates, frees, synchronises or calls NCCL; every kernel goes on `stream` (a cudaStream_t,
 *     NULL = the legacy default stream).  Calls are reentrant across streams.  The only global state is the
 *     row schedulers' per-launch counter slots (see echo_policy_loss_fwd_bwd) and cached per-device launch
 *     attributes.
 *   - The returned echo_status covers ARGUMENTS only (null pointers, sizes, alignment, device is not
 *     sm_100) and launch failures (cudaGetLastError -> ECHO_ERR_CUDA).  Data-dependent errors are
 *     reported on the device (echo_pack_result.status, the non-finite counter of echo_loss_stats) so
 *     that no call hides a host synchronisation.
 *   - Results are deterministic: no floating-point atomics; every reduction has a fixed order that
 *     depends only on the sizes (vocab, n_tokens), never on grid size, micro-batch split or rank.
 *   - Requires an sm_100 (B200) device; there is no fallback path.
 *
 * Environment: the GEMM, LM-head and f1 kernels read a few ECHO_* variables at launch (unit shapes, raster groups, L2
 * policies, ring shapes; DESIGN.md §7 "A/B knobs") so that the measurement tools can compare designs in one
 * process.  They are not part of this ABI and change results only within fp32 rounding (summation order); unset,
 * each takes its measured-best default.
 */
#ifndef ECHO_H
#define ECHO_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ECHO_API __attribute__((visibility("default")))
#else
#define ECHO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ECHO_OK = 0,
  ECHO_ERR_INVALID_ARGUMENT = 1,
  ECHO_ERR_UNSUPPORTED = 2, /* no sm_100 device / shape outside the kernels' range */
  ECHO_ERR_CUDA = 3         /* a CUDA runtime call or kernel launch failed */
} echo_status;

typedef enum { ECHO_F32 = 0, ECHO_BF16 = 1 } echo_dtype;

/* Data-dependent errors, written by echo_pack_batch into echo_pack_result.status. */
enum {
  ECHO_DATA_OK = 0,
  ECHO_DATA_FUTURE_VERSION = 1,      /* param_version > t_train (SPEC.md :388 t_infer <= t_train)     */
  ECHO_DATA_MIXED_GROUP_VERSION = 2, /* versions differ inside one prompt group (SPEC.md :48)          */
  ECHO_DATA_BAD_LENGTH = 3,          /* resp_len not in [1, max_len] (SPEC.md :39: length >= 1)        */
  ECHO_DATA_BAD_ACTION = 4,          /* a kept token's action not in [0, vocab)                        */
  ECHO_DATA_CAPACITY = 5             /* n_tokens > token_capacity: token arrays were not written       */
};

/* Per-token flag bits (tok_flags). */
enum { ECHO_FLAG_CLIPPED = 1, ECHO_FLAG_NONFINITE = 2 };

/* Algorithm selector for echo_policy_loss_fwd_bwd_ex (tests / benchmarks). */
enum {
  ECHO_ALGO_AUTO = 0,           /* OCT_REG for bf16 with 16384 <= vocab <= 155648, HEX_REG for bf16 up to
                                   311296 and for fp32 up to 155648, ROW_L2 otherwise */
  ECHO_ALGO_ROW_L2 = 1,         /* one 1024-thread CTA per row, two streaming passes, the second re-reads the row
                                   from L2; bf16 or fp32, any vocab */
  ECHO_ALGO_QUAD_REG = 2,       /* 4-CTA cluster per row, each CTA a quarter-row in registers, two CTAs (two rows)
                                   per SM, TMA-fed ring, DSMEM merge; exp(z - m) kept as fp16 between the passes
                                   (bf16, vocab <= 155648) -- the B200 design */
  ECHO_ALGO_QUAD_REG_EXACT = 3, /* as QUAD_REG, but the write-back recomputes exp from the bf16 logits (fp32 end to
                                   end; two exponentials per logit) */
  ECHO_ALGO_OCT_REG = 4,        /* as QUAD_REG with an 8-CTA cluster per row (eighth-rows in registers) and four
                                   CTAs (four rows) per SM; the fastest on B200 for Qwen vocabularies */
  ECHO_ALGO_HEX_REG = 5         /* as OCT_REG with a 16-CTA cluster (non-portable cluster size): bf16 vocabularies
                                   up to 311296 (Gemma / Llama-4 class), fp32 logits up to 155648 (the exps are
                                   kept at full fp32 precision between the passes) */
};

/* Device-resident result of echo_pack_batch (32 bytes). */
typedef struct {
  int32_t status;            /* ECHO_DATA_*                                                        */
  int32_t first_bad_rollout; /* global rollout id of the first error, -1 if none / CAPACITY          */
  int32_t n_groups_kept;
  int32_t n_rollouts_kept;   /* = n_groups_kept * group_size                                       */
  int64_t n_tokens;          /* packed (kept) tokens N_local = sum of kept resp_len                 */
  int64_t internal;          /* library scratch; do not read or write                              */
} echo_pack_result;

/*
 * (1) Version-lag filter + pack.
 * Cites: rollouts carry a param_version tag (PAPER.md :192); the coordinator bounds the policy lag by
 * the strict trigger t_train - t_infer > Delta_max (PAPER.md :224), so a rollout group is KEPT iff
 * t_train - version <= max_lag and dropped iff the lag is strictly greater -- the same predicate as the
 * buffer's param_version >= min_version (SPEC.md :344) with min_version = t_train - max_lag.
 *
 * Input layout (this rank's shard of the step's batch; group-major, SPEC.md :44-49):
 *   n_rollouts R (multiple of group_size), group_size G >= 2, max_len S >= 1, vocab V >= 1.
 *   version[R] int64, resp_len[R] int32; action / old_logp / ref_logp are padded row-major [R x S]
 *   (position j of rollout i at i*S + j; positions >= resp_len[i] are never read).  ref_logp may be
 *   NULL (then tok_ref must be NULL too).  aux [R x S] is an optional per-token payload packed like old_logp
 *   into tok_aux (e.g. the PPO-GAE advantages of echo_gae_advantage; both NULL or both set).
 *   rollout_base = global id of local rollout 0; it must be a multiple of group_size (a shard holds whole
 *   groups: pack groups rollouts by local index and echo_group_advantage by global id / G), else
 *   ECHO_ERR_INVALID_ARGUMENT.
 * Outputs (ascending, stable compaction; tokens rollout-major):
 *   kept_rollout[R]   global ids of kept rollouts (first n_rollouts_kept entries written)
 *   kept_offset[R+1]  CSR offsets into the token arrays (first n_rollouts_kept + 1 entries written)
 *   tok_slot / tok_action / tok_old / tok_ref [token_capacity]: per packed token its kept-rollout
 *   slot, action, old log-prob (the rollout's "logprobs" field, PAPER.md :162) and reference log-prob.
 *   *result (device): see echo_pack_result.  On a data error only status and first_bad_rollout are
 *   specified; the first error is the (rollout, check) lexicographic minimum with checks ordered
 *   FUTURE < MIXED < BAD_LENGTH < BAD_ACTION; CAPACITY only when no other error occurred.
 * Launches: 3 kernels.  Integer / bit-copy work only: results are bit-exact.
 */
ECHO_API echo_status echo_pack_batch(int32_t n_rollouts, int32_t group_size, int32_t max_len, int32_t vocab,
                                     int64_t t_train, int32_t max_lag, int64_t rollout_base,
                                     const int64_t* version, const int32_t* resp_len,
                                     const int32_t* action, const float* old_logp, const float* ref_logp,
                                     const float* aux, int64_t token_capacity,
                                     int32_t* kept_rollout, int64_t* kept_offset,
                                     int32_t* tok_slot, int32_t* tok_action, float* tok_old, float* tok_ref,
                                     float* tok_aux, echo_pack_result* result, void* stream);

/*
 * f3 ("partial-group handling if per-rollout versions ever differ"): echo_pack_batch with a
 * filter mode.  ECHO_FILTER_GROUP is echo_pack_batch (one decision per group from its uniform version;
 * MIXED_GROUP_VERSION otherwise).  ECHO_FILTER_ROLLOUT keeps rollout i iff t_train - version[i] <= max_lag, so a
 * group may keep only some of its rollouts: no MIXED check, n_groups_kept counts the groups with at least one
 * kept rollout, and echo_group_advantage normalises each group over its survivors.  Same outputs and launches.
 */
enum { ECHO_FILTER_GROUP = 0, ECHO_FILTER_ROLLOUT = 1 };
ECHO_API echo_status echo_pack_batch_v2(int32_t n_rollouts, int32_t group_size, int32_t max_len, int32_t vocab,
                                        int64_t t_train, int32_t max_lag, int64_t rollout_base,
                                        const int64_t* version, const int32_t* resp_len,
                                        const int32_t* action, const float* old_logp, const float* ref_logp,
                                        const float* aux, int64_t token_capacity,
                                        int32_t* kept_rollout, int64_t* kept_offset,
                                        int32_t* tok_slot, int32_t* tok_action, float* tok_old, float* tok_ref,
                                        float* tok_aux, echo_pack_result* result, int32_t filter_mode, void* stream);

/*
 * f4: PPO-GAE advantages over the per-step `rewards` and `values` of each trajectory (PAPER.md
 * :163-164, the fields "required by PPO and its popular variants", :170-171).  For rollout i, t = L_i-1 .. 0:
 *   delta_t = r_t + gamma V_{t+1} - V_t   (V_{L_i} = bootstrap_value[i]; 0 when bootstrap_value is NULL, i.e.
 *                                          terminal trajectories)
 *   A_t = delta_t + gamma lambda A_{t+1}  (A_{L_i} = 0);   returns_t = A_t + V_t   (returns nullable)
 * rewards / values / adv / returns are padded row-major [R x S]; positions >= resp_len[i] are neither read nor
 * written.  fp64 with round-to-nearest, no contraction, in this order: bit-identical to a sequential fp64 loop.
 * Launches: 1 kernel.
 */
ECHO_API echo_status echo_gae_advantage(int32_t n_rollouts, int32_t max_len, const int32_t* resp_len,
                                        const float* rewards, const float* values, const float* bootstrap_value,
                                        float gamma, float lam, float* adv, float* returns, void* stream);

/*
 * (2) GRPO group-relative advantage (PAPER.md :374 names GRPO; formula SPEC.md :209-213):
 *   for each kept group -- the run of consecutive kept rollouts with the same global id / G: G rollouts, or its
 *   n_g surviving rollouts after the per-rollout filter of echo_pack_batch_v2 -- in fp64 with round-to-nearest
 *   and no FMA contraction:
 *   mean = (sum r)/n_g, std = sqrt(sum (r - mean)^2 / n_g) (population), A = (r - mean)/(std + eps),
 *   rounded to fp32.  Every token of rollout i receives A_i through tok_slot (SPEC.md :209).
 * reward[R]: per-rollout return (sum of its per-step rewards, PAPER.md :164), indexed by local id.
 * kept_rollout / pack: outputs of echo_pack_batch on the same shard; rollout_base the same value as there (a
 *   multiple of group_size, else ECHO_ERR_INVALID_ARGUMENT).
 * Outputs: adv_slot[R] (first n_rollouts_kept written), adv_stats[6] fp64 partial sums
 *   {sum A, sum A^2, sum r, sum r^2, n_zero_std_groups, n_rollouts_kept} (A as fp32 values; per-group
 *   partials summed in ascending group order).  Bit-identical to a sequential fp64 evaluation.
 * Launches: 1 kernel.
 */
ECHO_API echo_status echo_group_advantage(int32_t n_rollouts, int32_t group_size, float eps,
                                 const float* reward, const int32_t* kept_rollout, int64_t rollout_base,
                                 const echo_pack_result* pack, float* adv_slot, double* adv_stats,
                                 void* stream);

/*
 * (3)+(4)+(5) fused: one streaming pass per logits row.
 *   (3) logp_t = z[t,a_t] - logsumexp_v z[t,v]   (the log pi_theta(a|s) field, PAPER.md :170)
 *   (4) rho = exp(logp - old); pg = max(-A rho, -A clip(rho, 1-clip_low, 1+clip_high)) (SPEC.md :219,
 *       eps 0.2 :243); if kl_coef > 0: kl = exp(ref-logp) - (ref-logp) - 1 (k3 to pi_ref);
 *       l_t = pg + kl_coef * kl;  the step loss is sum_t l_t / N_global.
 *   (5) c_t = grad_scale/N_global * ([not clipped](-A rho) + kl_coef (1 - exp(ref - logp)));
 *       logits[t, v] <- c_t (delta_{v,a_t} - softmax(z[t,:])_v)  for v < vocab (IN PLACE; columns
 *       vocab..ld-1 untouched).  "clipped" = (A > 0 and rho > 1+clip_high) or (A < 0 and rho < 1-clip_low).
 * logits: [n_rows x ld] row-major, dtype ECHO_BF16 or ECHO_F32, base and ld*sizeof(dtype) 16-byte
 *   aligned; row t is packed token t of this micro-batch.  Per-token inputs (tok_action, tok_old,
 *   tok_ref, tok_slot) are offset by the caller to the micro-batch's first row; tok_ref may be NULL iff
 *   kl_coef == 0.  adv_slot: echo_group_advantage output.  n_global: DEVICE pointer to one double,
 *   the all-reduced kept-token count (fed on device: no host sync).
 * Outputs per row: tok_logp, tok_loss (l_t, fp32), tok_flags (ECHO_FLAG_*).  A row whose lse, logp, rho,
 *   l_t or c_t is not finite gets ECHO_FLAG_NONFINITE; its gradient row is unspecified.
 * Arithmetic: fp32 accumulation over the bf16/fp32 logits, gradient stored with round-to-nearest-even.
 *   Deterministic: a row's reduction order depends only on vocab and the kernel, never on the grid, the stream,
 *   the micro-batch split or which cluster the row is scheduled on.
 * Concurrency: the kernels hand rows out from a per-launch counter slot (256 slots, each reset by its launch's last
 *   CTA).  Eager launches take slots 0..191 round robin, so up to 192 may be in flight at once on different
 *   streams; launches captured into a CUDA graph keep their slot for the graph's lifetime and take slots 192..255,
 *   so a replay never shares a counter with an eager launch.  Unsupported (rows would be skipped or done twice,
 *   silently): replaying one graph concurrently with itself, or more than 64 captured launches running at once.
 * Launches: 1 kernel (0 when n_rows == 0).
 */
ECHO_API echo_status echo_policy_loss_fwd_bwd(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                     const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                                     const int32_t* tok_slot, const float* adv_slot, const double* n_global,
                                     float clip_low, float clip_high, float kl_coef, float grad_scale,
                                     float* tok_logp, float* tok_loss, uint8_t* tok_flags, void* stream);

/* Same, with an explicit ECHO_ALGO_* choice (ECHO_ERR_UNSUPPORTED if that kernel cannot take the shape). */
ECHO_API echo_status echo_policy_loss_fwd_bwd_ex(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                        const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                                        const int32_t* tok_slot, const float* adv_slot, const double* n_global,
                                        float clip_low, float clip_high, float kl_coef, float grad_scale,
                                        float* tok_logp, float* tok_loss, uint8_t* tok_flags, int32_t algo,
                                        void* stream);

/*
 * Forward-only token log-probs: logp_t = z[t,a_t] - logsumexp_v z[t,v] (PAPER.md :170), the
 * quantity a trainer recomputes for old_logp (the behaviour policy, PAPER.md :162) and for ref_logp (the KL
 * reference, PAPER.md :278).  Same layout rules as echo_policy_loss_fwd_bwd; the logits are only READ (one HBM
 * pass, half the traffic of the fused kernel).  tok_lse (per-row log-sum-exp) and tok_flags
 * (ECHO_FLAG_NONFINITE) are nullable.  Launches: 1 kernel (0 when n_rows == 0).
 */
ECHO_API echo_status echo_token_logp(const void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                     const int32_t* tok_action, float* tok_logp, float* tok_lse, uint8_t* tok_flags,
                                     void* stream);

/* f4 loss variants ("PPO, KL-constrained PPO, GRPO ... or emerging variants", PAPER.md :278). */
enum { ECHO_KL_K3 = 0, /* exp(ref - logp) - (ref - logp) - 1: unbiased, non-negative (the default, reading R5) */
       ECHO_KL_K1 = 1, /* logp - ref: the Schulman k1 estimator of KL(pi_theta || pi_ref), d/dlogp = +1. NOT the
                        * sign of SPEC.md :244's k1 (logprob_old - logprob_new, against pi_old): passing old_logp as
                        * tok_ref does not reproduce that term -- its gradient has the opposite sign.             */
       ECHO_KL_K2 = 2  /* (logp - ref)^2 / 2                                                                   */ };

typedef struct {
  float clip_low, clip_high; /* PPO ratio clip [1 - clip_low, 1 + clip_high] (SPEC.md :219, :243: 0.2 / 0.2)  */
  float clip_dual;           /* dual clip c > 1: for A < 0 the loss is capped at -A c (0 = off)              */
  float kl_coef;             /* beta (PAPER.md :376-382: 0.001 or 0)                                         */
  float grad_scale;          /* s: multiplies every gradient coefficient                                     */
  int32_t kl_estimator;      /* ECHO_KL_*                                                                    */
  float entropy_coef;        /* eta >= 0: entropy bonus, l_t -= eta H_t (0 = off)                            */
} echo_loss_config;

/*
 * General form of echo_policy_loss_fwd_bwd (which is this call with tok_adv = tok_weight = tok_entropy = NULL,
 * clip_dual = 0, kl_estimator = ECHO_KL_K3, entropy_coef = 0):
 *   A_t = tok_adv ? tok_adv[t] : adv_slot[tok_slot[t]]   -- per-token advantages, e.g. PPO-GAE (echo_gae_advantage)
 *   w_t = tok_weight ? tok_weight[t] : 1 / *n_global      -- per-token loss weights, e.g. sequence-mean aggregation
 *                                                           (w_t = 1 / (n_sequences L_i)); n_global may then be NULL
 *   c_t = grad_scale * w_t * dl_t/dlogp ; tok_loss[t] = l_t (unweighted); the step loss is sum_t w_t l_t.
 * Entropy bonus (entropy_coef = eta > 0): H_t = -sum_v p_v log p_v (masked -inf logits contribute 0),
 *   l_t = pg + beta kl - eta H_t, and d[t,v] = c_t (delta_{v,a} - p_v) + grad_scale w_t eta p_v (log p_v + H_t).
 *   tok_entropy (nullable, f32[n_rows]) receives H_t.  With eta > 0 or tok_entropy set, the kernel also keeps
 *   sum_v z_v e^{z_v - m} in pass 1 and recomputes p_v from the logits in pass 2 (fp32 end to end, one more
 *   exponential per logit); explicit QUAD_REG and QUAD_REG_EXACT both run the 4-CTA entropy variant.
 * cfg is a HOST pointer.  Same layout, launches and errors as echo_policy_loss_fwd_bwd, plus
 * ECHO_ERR_INVALID_ARGUMENT for entropy_coef < 0 or not finite.
 */
ECHO_API echo_status echo_policy_loss_fwd_bwd_v2(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab,
                                                 int64_t ld, const int32_t* tok_action, const float* tok_old,
                                                 const float* tok_ref, const int32_t* tok_slot, const float* adv_slot,
                                                 const float* tok_adv, const float* tok_weight, const double* n_global,
                                                 const echo_loss_config* cfg, float* tok_logp, float* tok_loss,
                                                 uint8_t* tok_flags, float* tok_entropy, int32_t algo, void* stream);

/* Launch shape echo_policy_loss_fwd_bwd_ex would use on the current device (no launch):
 * shape[5] = {resolved algo, grid CTAs, CTAs per cluster, threads per CTA, dynamic smem bytes}. */
ECHO_API echo_status echo_policy_loss_launch_shape(int32_t dtype, int64_t n_rows, int32_t vocab, int32_t algo,
                                                   int32_t* shape);

/*
 * Statistics of the per-token outputs over n_tokens packed tokens (all micro-batches of the step):
 *   loss_stats[11] = {sum l_t, sum (logp - old), sum k3(ref, logp) (0 if tok_ref NULL), n_clipped,
 *                     n_nonfinite, rho_min, rho_max, sum logp, n_tokens, sum rho, sum w_t l_t}
 *   evaluated in fp64 from the fp32 per-token values (rho = exp(logp - old), k3 = e^x - x - 1 with
 *   x = ref - logp); rho statistics over rows without ECHO_FLAG_NONFINITE (rho_min = +inf, rho_max = -inf
 *   when there are none); w_t = tok_weight[t] (nullable: 1).  The step loss is sum l_t / N_global, or
 *   sum w_t l_t with per-token weights (echo_policy_loss_fwd_bwd_v2).  Fixed-order fp64 reduction:
 *   bitwise reproducible for a given n_tokens.
 * workspace: device buffer of echo_loss_stats_workspace_bytes() bytes (no initialisation needed).
 * Launches: 2 kernels.
 */
ECHO_API size_t echo_loss_stats_workspace_bytes(void);
ECHO_API echo_status echo_loss_stats(int64_t n_tokens, const float* tok_loss, const float* tok_logp,
                                     const float* tok_old, const float* tok_ref, const float* tok_weight,
                                     const uint8_t* tok_flags, double* workspace, double* loss_stats, void* stream);

/*
 * f3: token-balanced resharding after the stale filter (PAPER.md :224 drops whole groups, so the
 * ranks' kept-token counts diverge; the data-parallel learners of PAPER.md :258-261 then wait for the busiest).
 * paper_2508_05387_b200/parallel.py moves whole kept rollouts between ranks (NCCL all-to-all of the packed arrays,
 * contiguous in global rollout order); the receiver rebuilds the CSR of echo_pack_batch from the received lengths:
 *   kept_offset[i] = sum_{j<i} max(lengths[j], 0),  kept_offset[n] = total;  tok_slot[t] = i for t in
 *   [kept_offset[i], kept_offset[i+1]).
 * lengths: device int32[n]; kept_offset: device int64[n+1]; tok_slot: device int32[total] (nullable: offsets
 * only).  Launches: 1 kernel (scan), +1 (fill) when n > 0 and tok_slot is set.  Bit-exact.
 */
ECHO_API echo_status echo_csr_from_lengths(int32_t n, const int32_t* lengths, int64_t* kept_offset,
                                           int32_t* tok_slot, void* stream);

/*
 * f3: the staleness histogram of a step (the per-step log's staleness_histogram, SPEC.md :604, and the buffer's
 * version_histogram, SPEC.md :373; staleness = t_train - param_version, PAPER.md :192, :224).  Same rollout inputs
 * and keep rule as echo_pack_batch_v2 with filter_mode (ECHO_FILTER_GROUP: a rollout is kept iff its group's first
 * version has t_train - v <= max_lag; ECHO_FILTER_ROLLOUT: iff its own version does):
 *   hist: device int64 [4][n_bins + 2] = {kept rollouts, dropped rollouts, kept tokens, dropped tokens} per bin;
 *   bin 0 counts future versions (lag < 0), bin 1 + lag for 0 <= lag < n_bins, bin n_bins + 1 older rollouts;
 *   tokens = min(max(resp_len, 0), max_len).  Every bin is written (no initialisation needed); integer counts,
 *   bit-exact.  1 <= n_bins <= 4096.  Launches: 1 kernel.
 */
ECHO_API echo_status echo_staleness_histogram(int32_t n_rollouts, int32_t group_size, int32_t max_len,
                                              int64_t t_train, int32_t max_lag, const int64_t* version,
                                              const int32_t* resp_len, int32_t n_bins, int64_t* hist,
                                              int32_t filter_mode, void* stream);

/*
 * f2: the LM head fused with (3), forward only.  The logits are the LM head's output
 * z[t, v] = sum_k hidden[t, k] weight[v, k] (the model's last projection; PAPER.md :254-261, the learner computes
 * log pi_theta(a|s) of PAPER.md :170 from them), and
 *   lse_t = logsumexp_v z[t, v],   logp_t = z[t, a_t] - lse_t      (NaN when a_t is outside [0, vocab))
 * are computed without materialising z: a tcgen05 tensor-core GEMM (bf16 inputs, fp32 accumulation in TMEM) whose
 * epilogue reduces each 128 x 256 logits tile to per-row partials, then an ordered merge (deterministic).
 * hidden: device bf16 [n_rows x d] row-major; weight: device bf16 [vocab x d] row-major; both 16-byte aligned,
 * d % 8 == 0.  tok_lse nullable.  tok_entropy (nullable): H_t = -sum_v p_v log p_v of the row (the f4 entropy),
 * from a third per-tile partial sum z e^{z - m}.  workspace: device buffer of echo_lmhead_workspace_bytes(n_rows,
 * vocab) bytes (12 B per row per 256 vocabulary columns + 4 B per row; no initialisation needed).
 * Launches: 2 kernels (0 when n_rows == 0).  ECHO_ERR_INVALID_ARGUMENT on bad sizes / pointers / alignment.
 */
ECHO_API size_t echo_lmhead_workspace_bytes(int64_t n_rows, int32_t vocab);
ECHO_API echo_status echo_lmhead_logp(const void* hidden, const void* weight, int64_t n_rows, int32_t d,
                                      int32_t vocab, const int32_t* tok_action, float* tok_logp, float* tok_lse,
                                      float* tok_entropy, void* workspace, void* stream);

/*
 * (4) from log-probs alone -- for paths that produce logp without the logits (f2's echo_lmhead_logp, f1): the
 * clipped surrogate, KL and entropy bonus of echo_policy_loss_fwd_bwd_v2 (PAPER.md :278, :376-382; SPEC.md :219,
 * :243) evaluated per token from tok_logp (and tok_entropy H_t when cfg->entropy_coef > 0), with the same fp32
 * scalar arithmetic as the fused kernels' row epilogue:
 *   rho = exp(logp - old); pg, dual clip, KL estimator as in echo_policy_loss_fwd_bwd_v2; l_t = pg + beta kl - eta H;
 *   tok_coef[t]  = c_t = grad_scale * w_t * dl_t/dlogp      (the (5) coefficient: dL/dz = c_t (delta - p) + ...)
 *   tok_ecoef[t] = e_t = grad_scale * w_t * eta              (nullable; the entropy term's factor)
 *   w_t = tok_weight ? tok_weight[t] : 1 / *n_global.
 * All arrays are device f32[n_rows] (tok_flags u8) offset to the micro-batch; tok_ref needed iff kl_coef > 0,
 * tok_entropy iff entropy_coef > 0; cfg is a HOST pointer.  Launches: 1 kernel (0 when n_rows == 0).
 */
ECHO_API echo_status echo_loss_from_logp(int64_t n_rows, const float* tok_logp, const float* tok_entropy,
                                         const float* tok_old, const float* tok_ref, const int32_t* tok_slot,
                                         const float* adv_slot, const float* tok_adv, const float* tok_weight,
                                         const double* n_global, const echo_loss_config* cfg, float* tok_loss,
                                         uint8_t* tok_flags, float* tok_coef, float* tok_ecoef, void* stream);

/*
 * f2 backward, step 1 ("backward recomputes"): the logits gradient (5) of the LM head's output
 * z = hidden weight^T, recomputed tile by tile on the tcgen05 tensor cores (the GEMM of echo_lmhead_logp) instead of
 * being read back from a stored [n_rows x vocab] logits matrix:
 *   p[t, v] = exp(z[t, v] - tok_lse[t]),
 *   D[t, v] = tok_coef[t] (delta_{v, a_t} - p) + tok_ecoef[t] p (z[t, v] - tok_lse[t] + tok_entropy[t])
 * (the (5) row of echo_policy_loss_fwd_bwd_v2; PAPER.md :254-256), stored as bf16 (round to nearest even) into
 * dlogits [n_rows x ld] row-major, columns vocab..ld-1 untouched.  tok_lse / tok_entropy: echo_lmhead_logp outputs;
 * tok_coef / tok_ecoef: echo_loss_from_logp outputs (tok_ecoef nullable: no entropy term; tok_entropy read iff
 * tok_ecoef is set).  hidden / weight as echo_lmhead_logp; ld % 8 == 0, dlogits 16-byte aligned.
 * Launches: 1 kernel (0 when n_rows == 0).
 */
ECHO_API echo_status echo_lmhead_dlogits(const void* hidden, const void* weight, int64_t n_rows, int32_t d,
                                         int32_t vocab, const int32_t* tok_action, const float* tok_lse,
                                         const float* tok_coef, const float* tok_ecoef, const float* tok_entropy,
                                         void* dlogits, int64_t ld, void* stream);

/*
 * f2 backward ("backward recomputes to give dhidden and dW"; PAPER.md :254-261, the learner
 * computes the gradients of the policy): for chunks of chunk_rows tokens,
 *   D_chunk = echo_lmhead_dlogits(...) into dlogits_ws (bf16 [chunk_rows x ld], ld = vocab rounded up to 8)
 *   dhidden[chunk] = D_chunk weight            (f32 [n_rows x d], overwritten)
 *   dweight       (+)= D_chunk^T hidden[chunk] (f32 [vocab x d]; accumulate = 0 overwrites, 1 adds to it)
 * The two products are bf16 GEMMs with fp32 accumulation on this library's tcgen05 GEMM (echo_gemm_bf16: 2-CTA
 * UMMA with multicast 4-CTA clusters, K-major D / MN-major W for dhidden, MN-major D and hidden for dweight, the
 * output written by TMA stores or added in L2).  Deterministic for a fixed chunk_rows.  Launches: per chunk 3
 * kernels.  With n_rows == 0: dweight zeroed (accumulate = 0) or untouched.
 */
ECHO_API echo_status echo_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d,
                                          int32_t vocab, const int32_t* tok_action, const float* tok_lse,
                                          const float* tok_coef, const float* tok_ecoef, const float* tok_entropy,
                                          float* dhidden, float* dweight, int32_t accumulate, void* dlogits_ws,
                                          int64_t chunk_rows, void* stream);

/*
 * f2: the LM head's logits z[t, v] = sum_k hidden[t, k] weight[v, k] as a plain tcgen05 GEMM (the GEMM of
 * echo_lmhead_logp, fp32 accumulation in TMEM) stored as bf16 (round to nearest even) into logits [n_rows x ld]
 * row-major, columns vocab..ld-1 untouched; ld % 8 == 0, logits 16-byte aligned.  Launches: 1 kernel.
 */
ECHO_API echo_status echo_lmhead_logits(const void* hidden, const void* weight, int64_t n_rows, int32_t d,
                                        int32_t vocab, void* logits, int64_t ld, void* stream);

/*
 * f2 training step through the LM head, chunked (PAPER.md :254-261): for each chunk of
 * chunk_rows tokens,
 *   echo_lmhead_logits into logits_ws (bf16 [chunk_rows x ld], ld = vocab rounded up to 8),
 *   echo_policy_loss_fwd_bwd_v2 on that chunk ((3)-(5): tok_logp / tok_loss / tok_flags / tok_entropy of the
 *     chunk's tokens, the chunk becomes dL/dz in place),
 *   dhidden[chunk] = D weight, dweight (+)= D^T hidden[chunk]  (the tcgen05 GEMMs of echo_lmhead_backward).
 * Per-token arrays are full-length (offset per chunk by the library); arguments as echo_policy_loss_fwd_bwd_v2 and
 * echo_lmhead_backward.  The logits are the bf16 rounding of the fp32-accumulated z (a bf16 model's LM-head output).
 * Launches: per chunk 4 kernels.
 */
ECHO_API echo_status echo_lmhead_policy_loss_fwd_bwd(
    const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab, const int32_t* tok_action,
    const float* tok_old, const float* tok_ref, const int32_t* tok_slot, const float* adv_slot, const float* tok_adv,
    const float* tok_weight, const double* n_global, const echo_loss_config* cfg, float* tok_logp, float* tok_loss,
    uint8_t* tok_flags, float* tok_entropy, float* dhidden, float* dweight, int32_t accumulate, void* logits_ws,
    int64_t chunk_rows, void* stream);

/*
 * The tcgen05 GEMM behind echo_lmhead_backward (f2), exposed as a building block: c[m, n] (+)= sum_k A(m, k) B(n, k),
 * fp32 accumulation and output.  A(m, k) = a[m * lda + k] (a_mn = 0, K-major) or a[k * lda + m] (a_mn = 1, MN-major);
 * B(n, k) = b[n * ldb + k] (b_mn = 0) or b[k * ldb + n] (b_mn = 1); bf16 a, b 16-byte aligned with lda, ldb multiples
 * of 8 elements; c fp32 [m x ldc] row-major, accumulate = 1 adds to it.  So dhidden = D W is (a = D, a_mn 0, b = W,
 * b_mn 1) and dweight = D^T h is (a = D, a_mn 1, b = h, b_mn 1).  Launches: 1 kernel (0 when m or n is 0).
 */
ECHO_API echo_status echo_gemm_bf16(const void* a, int32_t a_mn, int64_t lda, const void* b, int32_t b_mn,
                                    int64_t ldb, int64_t m, int32_t n, int32_t k, float* c, int64_t ldc,
                                    int32_t accumulate, void* stream);

/* Human-readable name of a status code (static storage). */
ECHO_API const char* echo_status_string(echo_status status);

/* ABI version: bumped on any signature change. */
ECHO_API int32_t echo_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ECHO_H */
