// abi.cu -- the extern "C" entry points of libecho (include/echo.h): argument validation + launches.
#include <cfloat>

#include <cuda_bf16.h>

#include <stdlib.h>

#include "echo_internal.h"

namespace {

// sm_100 check + SM count of the current device (queried per call: no global mutable state).
echo_status device_sms(int* num_sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return ECHO_ERR_CUDA;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return ECHO_ERR_CUDA;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return ECHO_ERR_CUDA;
  if (major != 10 || minor != 0) return ECHO_ERR_UNSUPPORTED;
  if (cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return ECHO_ERR_CUDA;
  return ECHO_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

echo_status from_cuda(cudaError_t e) { return e == cudaSuccess ? ECHO_OK : ECHO_ERR_CUDA; }

// ECHO_ALGO_AUTO -> the 8-CTA register-resident kernel for bf16 Qwen-size vocabularies (2.91 ms vs 2.94 ms for the
// 4-CTA one on 32768 x 151936, profiles/), the row kernel otherwise; explicit choices are checked for support.
echo_status resolve_algo(int32_t dtype, int32_t vocab, int32_t* algo) {
  if (*algo < ECHO_ALGO_AUTO || *algo > ECHO_ALGO_HEX_REG) return ECHO_ERR_INVALID_ARGUMENT;
  const bool quad_ok = echo::quad_supports(dtype, vocab);
  if (*algo == ECHO_ALGO_AUTO)
    *algo = (echo::oct_supports(dtype, vocab) && vocab >= 16384) ? ECHO_ALGO_OCT_REG
            : echo::hex_supports(dtype, vocab) && vocab >= 16384 ? ECHO_ALGO_HEX_REG
                                                                  : ECHO_ALGO_ROW_L2;
  if ((*algo == ECHO_ALGO_QUAD_REG || *algo == ECHO_ALGO_QUAD_REG_EXACT) && !quad_ok) return ECHO_ERR_UNSUPPORTED;
  if (*algo == ECHO_ALGO_OCT_REG && !echo::oct_supports(dtype, vocab)) return ECHO_ERR_UNSUPPORTED;
  if (*algo == ECHO_ALGO_HEX_REG && !echo::hex_supports(dtype, vocab)) return ECHO_ERR_UNSUPPORTED;
  return ECHO_OK;
}

}  // namespace

#ifdef ECHO_TRACE
// Diagnostic build only (libecho_trace.so, tools/trace_kernel.py): per-CTA phase timestamps of the next calls.
static unsigned long long* g_trace = nullptr;
static int32_t g_trace_rows = 0;
extern "C" ECHO_API void echo_trace_set(unsigned long long* buf, int32_t rows) {
  g_trace = buf;
  g_trace_rows = rows;
}
#endif

extern "C" {

int32_t echo_abi_version(void) { return 4; }  // 4: the f2 backward lost its cuBLAS handle

const char* echo_status_string(echo_status s) {
  switch (s) {
    case ECHO_OK: return "ECHO_OK";
    case ECHO_ERR_INVALID_ARGUMENT: return "ECHO_ERR_INVALID_ARGUMENT";
    case ECHO_ERR_UNSUPPORTED: return "ECHO_ERR_UNSUPPORTED";
    case ECHO_ERR_CUDA: return "ECHO_ERR_CUDA";
  }
  return "ECHO_ERR_UNKNOWN";
}

echo_status echo_pack_batch(int32_t n_rollouts, int32_t group_size, int32_t max_len, int32_t vocab, int64_t t_train,
                            int32_t max_lag, int64_t rollout_base, const int64_t* version, const int32_t* resp_len,
                            const int32_t* action, const float* old_logp, const float* ref_logp, const float* aux,
                            int64_t token_capacity, int32_t* kept_rollout, int64_t* kept_offset, int32_t* tok_slot,
                            int32_t* tok_action, float* tok_old, float* tok_ref, float* tok_aux,
                            echo_pack_result* result, void* stream) {
  return echo_pack_batch_v2(n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, version, resp_len,
                            action, old_logp, ref_logp, aux, token_capacity, kept_rollout, kept_offset, tok_slot,
                            tok_action, tok_old, tok_ref, tok_aux, result, ECHO_FILTER_GROUP, stream);
}

echo_status echo_pack_batch_v2(int32_t n_rollouts, int32_t group_size, int32_t max_len, int32_t vocab,
                               int64_t t_train, int32_t max_lag, int64_t rollout_base, const int64_t* version,
                               const int32_t* resp_len, const int32_t* action, const float* old_logp,
                               const float* ref_logp, const float* aux, int64_t token_capacity, int32_t* kept_rollout,
                               int64_t* kept_offset, int32_t* tok_slot, int32_t* tok_action, float* tok_old,
                               float* tok_ref, float* tok_aux, echo_pack_result* result, int32_t filter_mode,
                               void* stream) {
  if (n_rollouts < 0 || group_size < 2 || max_len < 1 || vocab < 1 || max_lag < 0 || token_capacity < 0)
    return ECHO_ERR_INVALID_ARGUMENT;
  if (filter_mode != ECHO_FILTER_GROUP && filter_mode != ECHO_FILTER_ROLLOUT) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rollouts % group_size != 0) return ECHO_ERR_INVALID_ARGUMENT;
  if (rollout_base < 0 || rollout_base + (int64_t)n_rollouts > INT32_MAX) return ECHO_ERR_INVALID_ARGUMENT;
  // pack groups rollouts by local index, (2) by global id / G: the two agree only on a group boundary
  if (rollout_base % group_size != 0) return ECHO_ERR_INVALID_ARGUMENT;
  if (!result || !kept_offset || (n_rollouts > 0 && (!version || !resp_len || !action || !old_logp || !kept_rollout)))
    return ECHO_ERR_INVALID_ARGUMENT;
  if (token_capacity > 0 && (!tok_slot || !tok_action || !tok_old)) return ECHO_ERR_INVALID_ARGUMENT;
  if ((ref_logp == nullptr) != (tok_ref == nullptr)) return ECHO_ERR_INVALID_ARGUMENT;
  if ((aux == nullptr) != (tok_aux == nullptr)) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_pack(n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, version,
                                     resp_len, action, old_logp, ref_logp, aux, token_capacity, kept_rollout,
                                     kept_offset, tok_slot, tok_action, tok_old, tok_ref, tok_aux, result,
                                     static_cast<cudaStream_t>(stream), sms, filter_mode));
}

echo_status echo_gae_advantage(int32_t n_rollouts, int32_t max_len, const int32_t* resp_len, const float* rewards,
                               const float* values, const float* bootstrap_value, float gamma, float lam, float* adv,
                               float* returns, void* stream) {
  if (n_rollouts < 0 || max_len < 1 || !(gamma >= 0.0f && gamma <= 1.0f) || !(lam >= 0.0f && lam <= 1.0f))
    return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rollouts > 0 && (!resp_len || !rewards || !values || !adv)) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_gae(n_rollouts, max_len, resp_len, rewards, values, bootstrap_value, gamma, lam, adv,
                                    returns, static_cast<cudaStream_t>(stream)));
}

echo_status echo_group_advantage(int32_t n_rollouts, int32_t group_size, float eps, const float* reward,
                                 const int32_t* kept_rollout, int64_t rollout_base, const echo_pack_result* pack,
                                 float* adv_slot, double* adv_stats, void* stream) {
  if (n_rollouts < 0 || group_size < 2 || n_rollouts % group_size != 0 || !(eps >= 0.0f))
    return ECHO_ERR_INVALID_ARGUMENT;
  if (rollout_base < 0 || rollout_base % group_size != 0) return ECHO_ERR_INVALID_ARGUMENT;
  if (!pack || !adv_stats || (n_rollouts > 0 && (!reward || !kept_rollout || !adv_slot)))
    return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_group_advantage(group_size, eps, rollout_base, reward, kept_rollout, pack, adv_slot,
                                                adv_stats, static_cast<cudaStream_t>(stream)));
}

echo_status echo_policy_loss_fwd_bwd_v2(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                        const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                                        const int32_t* tok_slot, const float* adv_slot, const float* tok_adv,
                                        const float* tok_weight, const double* n_global, const echo_loss_config* cfg,
                                        float* tok_logp, float* tok_loss, uint8_t* tok_flags, float* tok_entropy,
                                        int32_t algo, void* stream) {
  if (!cfg) return ECHO_ERR_INVALID_ARGUMENT;
  if (dtype != ECHO_F32 && dtype != ECHO_BF16) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows < 0 || vocab < 1 || ld < vocab) return ECHO_ERR_INVALID_ARGUMENT;
  const int64_t esize = dtype == ECHO_BF16 ? 2 : 4;
  if ((ld * esize) % 16 != 0) return ECHO_ERR_INVALID_ARGUMENT;
  if (!(cfg->clip_low >= 0.0f && cfg->clip_low < 1.0f && cfg->clip_high >= 0.0f) || !(cfg->kl_coef >= 0.0f) ||
      !(cfg->clip_dual == 0.0f || cfg->clip_dual > 1.0f) || cfg->kl_estimator < ECHO_KL_K3 ||
      cfg->kl_estimator > ECHO_KL_K2 || !(cfg->entropy_coef >= 0.0f && cfg->entropy_coef <= FLT_MAX))
    return ECHO_ERR_INVALID_ARGUMENT;
  if (!n_global && !tok_weight) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0) {
    if (!logits || !aligned16(logits) || !tok_action || !tok_old || !tok_logp || !tok_loss || !tok_flags)
      return ECHO_ERR_INVALID_ARGUMENT;
    if (!tok_adv && (!tok_slot || !adv_slot)) return ECHO_ERR_INVALID_ARGUMENT;
    if (cfg->kl_coef > 0.0f && !tok_ref) return ECHO_ERR_INVALID_ARGUMENT;
  }
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  if (n_rows == 0) return ECHO_OK;
  st = resolve_algo(dtype, vocab, &algo);
  if (st != ECHO_OK) return st;
  echo::LossParams p{};
  p.logits = static_cast<uint8_t*>(logits);
  p.n_rows = n_rows;
  p.V = vocab;
  p.ld_bytes = ld * esize;
  p.tok_action = tok_action;
  p.tok_old = tok_old;
  p.tok_ref = tok_ref;
  p.tok_slot = tok_slot;
  p.adv_slot = adv_slot;
  p.n_global = n_global;
  p.clip_low = cfg->clip_low;
  p.clip_high = cfg->clip_high;
  p.kl_coef = cfg->kl_coef;
  p.grad_scale = cfg->grad_scale;
  p.clip_dual = cfg->clip_dual;
  p.kl_estimator = cfg->kl_estimator;
  p.tok_adv = tok_adv;
  p.tok_weight = tok_weight;
  p.entropy_coef = cfg->entropy_coef;
  p.tok_entropy = tok_entropy;
  p.tok_logp = tok_logp;
  p.tok_loss = tok_loss;
  p.tok_flags = tok_flags;
  p.tok_lse = nullptr;
  p.trace = nullptr;
  p.trace_rows = 0;
#ifdef ECHO_TRACE
  p.trace = g_trace;
  p.trace_rows = g_trace_rows;
#endif
  return from_cuda(echo::launch_policy_loss(p, dtype, algo, static_cast<cudaStream_t>(stream), sms));
}

echo_status echo_policy_loss_fwd_bwd_ex(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                        const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                                        const int32_t* tok_slot, const float* adv_slot, const double* n_global,
                                        float clip_low, float clip_high, float kl_coef, float grad_scale,
                                        float* tok_logp, float* tok_loss, uint8_t* tok_flags, int32_t algo,
                                        void* stream) {
  if (!n_global) return ECHO_ERR_INVALID_ARGUMENT;
  const echo_loss_config cfg{clip_low, clip_high, 0.0f, kl_coef, grad_scale, ECHO_KL_K3, 0.0f};
  return echo_policy_loss_fwd_bwd_v2(logits, dtype, n_rows, vocab, ld, tok_action, tok_old, tok_ref, tok_slot,
                                     adv_slot, nullptr, nullptr, n_global, &cfg, tok_logp, tok_loss, tok_flags,
                                     nullptr, algo, stream);
}

echo_status echo_policy_loss_fwd_bwd(void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                                     const int32_t* tok_action, const float* tok_old, const float* tok_ref,
                                     const int32_t* tok_slot, const float* adv_slot, const double* n_global,
                                     float clip_low, float clip_high, float kl_coef, float grad_scale, float* tok_logp,
                                     float* tok_loss, uint8_t* tok_flags, void* stream) {
  return echo_policy_loss_fwd_bwd_ex(logits, dtype, n_rows, vocab, ld, tok_action, tok_old, tok_ref, tok_slot,
                                     adv_slot, n_global, clip_low, clip_high, kl_coef, grad_scale, tok_logp, tok_loss,
                                     tok_flags, ECHO_ALGO_AUTO, stream);
}

echo_status echo_policy_loss_launch_shape(int32_t dtype, int64_t n_rows, int32_t vocab, int32_t algo,
                                          int32_t* shape) {
  if ((dtype != ECHO_F32 && dtype != ECHO_BF16) || n_rows < 1 || vocab < 1 || !shape) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  st = resolve_algo(dtype, vocab, &algo);
  if (st != ECHO_OK) return st;
  echo::LossParams p{};
  p.n_rows = n_rows;
  p.V = vocab;
  echo::LaunchShape s{};
  st = from_cuda(echo::launch_policy_loss(p, dtype, algo, nullptr, sms, &s));
  if (st != ECHO_OK) return st;
  shape[0] = algo;
  shape[1] = s.grid_ctas;
  shape[2] = s.cluster_ctas;
  shape[3] = s.threads;
  shape[4] = s.smem_bytes;
  return ECHO_OK;
}

echo_status echo_token_logp(const void* logits, int32_t dtype, int64_t n_rows, int32_t vocab, int64_t ld,
                            const int32_t* tok_action, float* tok_logp, float* tok_lse, uint8_t* tok_flags,
                            void* stream) {
  if (dtype != ECHO_F32 && dtype != ECHO_BF16) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows < 0 || vocab < 1 || ld < vocab) return ECHO_ERR_INVALID_ARGUMENT;
  const int64_t esize = dtype == ECHO_BF16 ? 2 : 4;
  if ((ld * esize) % 16 != 0) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0 && (!logits || !aligned16(logits) || !tok_action || !tok_logp)) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  if (n_rows == 0) return ECHO_OK;
  echo::LossParams p{};
  p.logits = static_cast<uint8_t*>(const_cast<void*>(logits));  // read only in this mode
  p.n_rows = n_rows;
  p.V = vocab;
  p.ld_bytes = ld * esize;
  p.tok_action = tok_action;
  p.tok_logp = tok_logp;
  p.tok_lse = tok_lse;
  p.tok_flags = tok_flags;
  p.kl_coef = 0.0f;
#ifdef ECHO_TRACE
  p.trace = g_trace;
  p.trace_rows = g_trace_rows;
#endif
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  // bf16: one warp per row (token_logp.cu); ECHO_LOGP_CLUSTER=1 selects the fused kernel's cluster tile in logp mode
  const char* env = getenv("ECHO_LOGP_CLUSTER");
  const bool cluster = env && atoi(env) != 0;
  if (!cluster && echo::token_logp_warp_supports(dtype, vocab))
    return from_cuda(echo::launch_token_logp_warp(p, s, sms));
  if (echo::hex_supports(dtype, vocab) && vocab >= 16384)
    return from_cuda(echo::launch_quad_logp(p, dtype, s, sms, nullptr));
  return from_cuda(echo::launch_row(p, dtype, s, sms, nullptr, false));
}

echo_status echo_staleness_histogram(int32_t n_rollouts, int32_t group_size, int32_t max_len, int64_t t_train,
                                     int32_t max_lag, const int64_t* version, const int32_t* resp_len, int32_t n_bins,
                                     int64_t* hist, int32_t filter_mode, void* stream) {
  if (n_rollouts < 0 || group_size < 1 || n_rollouts % group_size != 0 || max_len < 1 || max_lag < 0 ||
      n_bins < 1 || n_bins > 4096 || !hist || (n_rollouts > 0 && (!version || !resp_len)) ||
      (filter_mode != ECHO_FILTER_GROUP && filter_mode != ECHO_FILTER_ROLLOUT))
    return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_staleness_hist(n_rollouts, group_size, max_len, t_train, max_lag, version, resp_len,
                                               n_bins, hist, filter_mode, static_cast<cudaStream_t>(stream)));
}

echo_status echo_csr_from_lengths(int32_t n, const int32_t* lengths, int64_t* kept_offset, int32_t* tok_slot,
                                  void* stream) {
  if (n < 0 || !kept_offset || (n > 0 && !lengths)) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_csr_from_lengths(n, lengths, kept_offset, tok_slot,
                                                 static_cast<cudaStream_t>(stream), sms));
}

size_t echo_lmhead_workspace_bytes(int64_t n_rows, int32_t vocab) {
  if (n_rows < 0 || vocab < 1) return 0;
  return echo::lmhead_workspace_bytes(n_rows, vocab);
}

echo_status echo_lmhead_logp(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab,
                             const int32_t* tok_action, float* tok_logp, float* tok_lse, float* tok_entropy,
                             void* workspace, void* stream) {
  if (n_rows < 0 || d < 8 || d % 8 != 0 || vocab < 1) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0 && (!hidden || !weight || !aligned16(hidden) || !aligned16(weight) || !tok_action || !tok_logp ||
                     !workspace))
    return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  if (n_rows == 0) return ECHO_OK;
  const cudaError_t e = echo::launch_lmhead_logp(hidden, weight, n_rows, d, vocab, tok_action, tok_logp, tok_lse,
                                                 tok_entropy, workspace, static_cast<cudaStream_t>(stream), sms);
  if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
  return from_cuda(e);
}

static bool valid_loss_config(const echo_loss_config* cfg) {
  return cfg && cfg->clip_low >= 0.0f && cfg->clip_low < 1.0f && cfg->clip_high >= 0.0f && cfg->kl_coef >= 0.0f &&
         (cfg->clip_dual == 0.0f || cfg->clip_dual > 1.0f) && cfg->kl_estimator >= ECHO_KL_K3 &&
         cfg->kl_estimator <= ECHO_KL_K2 && cfg->entropy_coef >= 0.0f && cfg->entropy_coef <= FLT_MAX;
}

echo_status echo_loss_from_logp(int64_t n_rows, const float* tok_logp, const float* tok_entropy, const float* tok_old,
                                const float* tok_ref, const int32_t* tok_slot, const float* adv_slot,
                                const float* tok_adv, const float* tok_weight, const double* n_global,
                                const echo_loss_config* cfg, float* tok_loss, uint8_t* tok_flags, float* tok_coef,
                                float* tok_ecoef, void* stream) {
  if (n_rows < 0 || !valid_loss_config(cfg)) return ECHO_ERR_INVALID_ARGUMENT;
  if (!n_global && !tok_weight) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0) {
    if (!tok_logp || !tok_old || !tok_loss || !tok_flags || !tok_coef) return ECHO_ERR_INVALID_ARGUMENT;
    if (!tok_adv && (!tok_slot || !adv_slot)) return ECHO_ERR_INVALID_ARGUMENT;
    if (cfg->kl_coef > 0.0f && !tok_ref) return ECHO_ERR_INVALID_ARGUMENT;
    if (cfg->entropy_coef > 0.0f && !tok_entropy) return ECHO_ERR_INVALID_ARGUMENT;
  }
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_loss_from_logp(n_rows, tok_logp, tok_entropy, tok_old, tok_ref, tok_slot, adv_slot,
                                               tok_adv, tok_weight, n_global, *cfg, tok_loss, tok_flags, tok_coef,
                                               tok_ecoef, static_cast<cudaStream_t>(stream), sms));
}

static bool valid_lmhead_shape(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab) {
  if (n_rows < 0 || d < 8 || d % 8 != 0 || vocab < 1) return false;
  return n_rows == 0 || (hidden && weight && aligned16(hidden) && aligned16(weight));
}

echo_status echo_lmhead_dlogits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab,
                                const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                const float* tok_ecoef, const float* tok_entropy, void* dlogits, int64_t ld,
                                void* stream) {
  if (!valid_lmhead_shape(hidden, weight, n_rows, d, vocab) || ld < vocab || ld % 8 != 0)
    return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0 && (!tok_action || !tok_lse || !tok_coef || !dlogits || !aligned16(dlogits) ||
                     (tok_ecoef && !tok_entropy)))
    return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  if (n_rows == 0) return ECHO_OK;
  const cudaError_t e = echo::launch_lmhead_dlogits(hidden, weight, n_rows, d, vocab, tok_action, tok_lse, tok_coef,
                                                    tok_ecoef, tok_entropy, dlogits, ld,
                                                    static_cast<cudaStream_t>(stream), sms);
  if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
  return from_cuda(e);
}

echo_status echo_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab,
                                 const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                 const float* tok_ecoef, const float* tok_entropy, float* dhidden, float* dweight,
                                 int32_t accumulate, void* dlogits_ws, int64_t chunk_rows, void* stream) {
  if (!valid_lmhead_shape(hidden, weight, n_rows, d, vocab) || chunk_rows < 1 || chunk_rows > INT32_MAX)
    return ECHO_ERR_INVALID_ARGUMENT;
  if (!dweight || (n_rows > 0 && (!tok_action || !tok_lse || !tok_coef || !dhidden || !dlogits_ws ||
                                  !aligned16(dlogits_ws) || (tok_ecoef && !tok_entropy))))
    return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  if (n_rows == 0) {
    if (accumulate) return ECHO_OK;
    return from_cuda(cudaMemsetAsync(dweight, 0, (size_t)vocab * d * sizeof(float), static_cast<cudaStream_t>(stream)));
  }
  const cudaError_t e = echo::launch_lmhead_backward(hidden, weight, n_rows, d, vocab, tok_action, tok_lse, tok_coef,
                                                     tok_ecoef, tok_entropy, dhidden, dweight, accumulate != 0,
                                                     dlogits_ws, chunk_rows, static_cast<cudaStream_t>(stream), sms);
  if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
  return from_cuda(e);
}

echo_status echo_lmhead_logits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t vocab,
                               void* logits, int64_t ld, void* stream) {
  if (!valid_lmhead_shape(hidden, weight, n_rows, d, vocab) || ld < vocab || ld % 8 != 0)
    return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0 && (!logits || !aligned16(logits))) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  const cudaError_t e = echo::launch_lmhead_logits(hidden, weight, n_rows, d, vocab, logits, ld,
                                                   static_cast<cudaStream_t>(stream), sms);
  if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
  return from_cuda(e);
}

echo_status echo_lmhead_policy_loss_fwd_bwd(const void* hidden, const void* weight, int64_t n_rows, int32_t d,
                                            int32_t vocab, const int32_t* tok_action, const float* tok_old,
                                            const float* tok_ref, const int32_t* tok_slot, const float* adv_slot,
                                            const float* tok_adv, const float* tok_weight, const double* n_global,
                                            const echo_loss_config* cfg, float* tok_logp, float* tok_loss,
                                            uint8_t* tok_flags, float* tok_entropy, float* dhidden, float* dweight,
                                            int32_t accumulate, void* logits_ws, int64_t chunk_rows,
                                            void* stream) {
  if (!valid_lmhead_shape(hidden, weight, n_rows, d, vocab) || chunk_rows < 1 || chunk_rows > INT32_MAX ||
      !dweight || !valid_loss_config(cfg))
    return ECHO_ERR_INVALID_ARGUMENT;
  if (n_rows > 0 && (!dhidden || !logits_ws || !aligned16(logits_ws))) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_rows == 0) return accumulate ? ECHO_OK : from_cuda(cudaMemsetAsync(dweight, 0, (size_t)vocab * d * 4, s));
  const int64_t ld = ((int64_t)vocab + 7) & ~(int64_t)7;
  const uint16_t* hid = static_cast<const uint16_t*>(hidden);
  for (int64_t r0 = 0; r0 < n_rows; r0 += chunk_rows) {
    const int64_t rows = (n_rows - r0 < chunk_rows) ? n_rows - r0 : chunk_rows;
    cudaError_t e = echo::launch_lmhead_logits(hid + r0 * d, weight, rows, d, vocab, logits_ws, ld, s, sms);
    if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
    if (e != cudaSuccess) return ECHO_ERR_CUDA;
    st = echo_policy_loss_fwd_bwd_v2(logits_ws, ECHO_BF16, rows, vocab, ld, tok_action + r0, tok_old + r0,
                                     tok_ref ? tok_ref + r0 : nullptr, tok_slot ? tok_slot + r0 : nullptr, adv_slot,
                                     tok_adv ? tok_adv + r0 : nullptr, tok_weight ? tok_weight + r0 : nullptr,
                                     n_global, cfg, tok_logp + r0, tok_loss + r0, tok_flags + r0,
                                     tok_entropy ? tok_entropy + r0 : nullptr, ECHO_ALGO_AUTO, stream);
    if (st != ECHO_OK) return st;
    e = echo::tc_lmhead_grads(s, sms, weight, hid + r0 * d, logits_ws, ld, rows, d, vocab, dhidden + r0 * d, dweight,
                              accumulate || r0 > 0);
    if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
    if (e != cudaSuccess) return ECHO_ERR_CUDA;
  }
  return from_cuda(cudaGetLastError());
}

echo_status echo_gemm_bf16(const void* a, int32_t a_mn, int64_t lda, const void* b, int32_t b_mn, int64_t ldb,
                           int64_t m, int32_t n, int32_t k, float* c, int64_t ldc, int32_t accumulate, void* stream) {
  if (m < 0 || n < 0 || k < 1 || m > INT32_MAX || lda < 1 || ldb < 1 || ldc < n || (lda * 2) % 16 || (ldb * 2) % 16)
    return ECHO_ERR_INVALID_ARGUMENT;
  if (lda < (a_mn ? m : k) || ldb < (b_mn ? n : k)) return ECHO_ERR_INVALID_ARGUMENT;
  if (m > 0 && n > 0 && (!a || !b || !c || !aligned16(a) || !aligned16(b))) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  const cudaError_t e = echo::gemm_bf16(a, a_mn != 0, lda * 2, b, b_mn != 0, ldb * 2, m, n, k, c, ldc, accumulate != 0,
                                        static_cast<cudaStream_t>(stream), sms);
  if (e == cudaErrorInvalidValue) return ECHO_ERR_INVALID_ARGUMENT;
  return from_cuda(e);
}

size_t echo_loss_stats_workspace_bytes(void) { return echo::loss_stats_workspace_bytes(); }

echo_status echo_loss_stats(int64_t n_tokens, const float* tok_loss, const float* tok_logp, const float* tok_old,
                            const float* tok_ref, const float* tok_weight, const uint8_t* tok_flags, double* workspace,
                            double* loss_stats, void* stream) {
  if (n_tokens < 0 || !workspace || !loss_stats) return ECHO_ERR_INVALID_ARGUMENT;
  if (n_tokens > 0 && (!tok_loss || !tok_logp || !tok_old || !tok_flags)) return ECHO_ERR_INVALID_ARGUMENT;
  int sms = 0;
  echo_status st = device_sms(&sms);
  if (st != ECHO_OK) return st;
  return from_cuda(echo::launch_loss_stats(n_tokens, tok_loss, tok_logp, tok_old, tok_ref, tok_weight, tok_flags,
                                           workspace, loss_stats, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
