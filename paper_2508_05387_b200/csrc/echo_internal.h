// echo_internal.h -- host-side launcher declarations shared by the libecho translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "echo.h"

#include <atomic>

namespace echo {

// Row / tile scheduler counter slot of one launch (each slot reset by its launch's last CTA).  Launches captured into
// a CUDA graph keep their slot for the graph's lifetime, so they draw from the top quarter of the slots and eager
// launches from the rest: an eager launch never shares a counter with a graph replay, whatever the launch count.
// Collisions remain possible only between more than n_slots / 4 captured launches replayed concurrently, or more
// than 3 n_slots / 4 eager launches in flight at once (include/echo.h "Concurrency").
inline uint32_t next_sched_slot(std::atomic<uint32_t>& eager, std::atomic<uint32_t>& captured, cudaStream_t stream,
                                uint32_t n_slots) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const uint32_t n_graph = n_slots / 4, n_eager = n_slots - n_graph;
  if (cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    return n_eager + captured.fetch_add(1, std::memory_order_relaxed) % n_graph;
  return eager.fetch_add(1, std::memory_order_relaxed) % n_eager;
}

// Parameter block of the fused policy-loss kernels (passed by value as a kernel argument).
struct LossParams {
  uint8_t* logits;
  int64_t n_rows;
  int32_t V;
  int64_t ld_bytes;
  const int32_t* __restrict__ tok_action;
  const float* __restrict__ tok_old;
  const float* __restrict__ tok_ref;
  const int32_t* __restrict__ tok_slot;
  const float* __restrict__ adv_slot;
  const double* __restrict__ n_global;
  float clip_low, clip_high, kl_coef, grad_scale;
  float clip_dual;                          // dual-clip constant c (> 1 enables), f4
  int32_t kl_estimator;                     // ECHO_KL_*, f4
  float entropy_coef;                       // eta: entropy bonus, f4
  float* __restrict__ tok_entropy;          // per-token entropy output (nullable), f4
  const float* __restrict__ tok_adv;        // per-token advantages (nullable: adv_slot[tok_slot])
  const float* __restrict__ tok_weight;     // per-token loss weights (nullable: 1 / N_global)
  float* __restrict__ tok_logp;
  float* __restrict__ tok_loss;
  uint8_t* __restrict__ tok_flags;
  float* __restrict__ tok_lse;  // forward-only mode (echo_token_logp): per-row log-sum-exp, nullable
  int32_t sched_slot;         // quad kernels: row-scheduler slot of this launch (set by the launcher)
  unsigned long long* trace;  // ECHO_TRACE builds only: per-CTA phase timestamps (tools/trace_kernel.py)
  int32_t trace_rows;
};

cudaError_t launch_pack(int32_t R, int32_t G, int32_t S, int32_t V, int64_t t_train, int32_t max_lag,
                        int64_t rollout_base, const int64_t* version, const int32_t* resp_len, const int32_t* action,
                        const float* old_logp, const float* ref_logp, const float* aux, int64_t cap,
                        int32_t* kept_rollout, int64_t* kept_offset, int32_t* tok_slot, int32_t* tok_action,
                        float* tok_old, float* tok_ref, float* tok_aux, echo_pack_result* res, cudaStream_t stream,
                        int num_sms, int32_t filter_mode = 0);

cudaError_t launch_group_advantage(int32_t G, float eps, int64_t rollout_base, const float* reward,
                                   const int32_t* kept_rollout, const echo_pack_result* pack, float* adv_slot,
                                   double* adv_stats, cudaStream_t stream);


// Launch shape a policy-loss call uses (reported by echo_policy_loss_launch_shape).
struct LaunchShape {
  int32_t grid_ctas, cluster_ctas, threads, smem_bytes;
};
// Per-kernel launchers (policy_loss_{quad,row}.cu); with shape != nullptr: report the shape, launch nothing.
cudaError_t launch_row(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms, LaunchShape* shape,
                       bool grad = true);
// f1: forward-only log-probs, one warp per row (token_logp.cu)
bool token_logp_warp_supports(int32_t dtype, int32_t V);
cudaError_t launch_token_logp_warp(const LossParams& p, cudaStream_t stream, int num_sms);
cudaError_t launch_quad_logp(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms,
                             LaunchShape* shape);
int max_active_clusters(const void* fn, int threads, size_t smem, int cluster, int fallback);
cudaError_t launch_quad(const LossParams& p, bool store_exp, cudaStream_t stream, int num_sms, LaunchShape* shape);
bool quad_supports(int32_t dtype, int32_t V);
bool oct_supports(int32_t dtype, int32_t V);
bool hex_supports(int32_t dtype, int32_t V);
cudaError_t launch_hex(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms, LaunchShape* shape);
cudaError_t launch_oct(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape);
// Dispatch by algorithm; with shape != nullptr: fill in the launch shape and launch nothing.
cudaError_t launch_policy_loss(const LossParams& p, int32_t dtype, int algo, cudaStream_t stream, int num_sms,
                               LaunchShape* shape = nullptr);

cudaError_t launch_gae(int32_t R, int32_t S, const int32_t* resp_len, const float* rewards, const float* values,
                       const float* bootstrap, float gamma, float lam, float* adv, float* ret, cudaStream_t stream);

cudaError_t launch_staleness_hist(int32_t R, int32_t G, int32_t S, int64_t t_train, int32_t max_lag,
                                  const int64_t* version, const int32_t* resp_len, int32_t n_bins, int64_t* hist,
                                  int32_t filter_mode, cudaStream_t stream);
cudaError_t launch_csr_from_lengths(int32_t n, const int32_t* lengths, int64_t* offsets, int32_t* tok_slot,
                                    cudaStream_t stream, int num_sms);

size_t lmhead_workspace_bytes(int64_t n_rows, int32_t V);
cudaError_t launch_lmhead_logp(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                               const int32_t* tok_action, float* tok_logp, float* tok_lse, float* tok_entropy,
                               void* workspace, cudaStream_t stream, int num_sms);

cudaError_t launch_lmhead_dlogits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                  const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                  const float* tok_ecoef, const float* tok_entropy, void* dlogits, int64_t ld,
                                  cudaStream_t stream, int num_sms);
cudaError_t launch_lmhead_logits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                 void* logits, int64_t ld, cudaStream_t stream, int num_sms);
// C[M x N] (+)= A B on the tcgen05 tensor cores (gemm.cu): A(m, k) from a K-major [M x K] (a_mn = false) or MN-major
// [K x M] (a_mn = true) bf16 array, B(n, k) likewise with N; row strides in bytes (multiples of 16); fp32 out.
cudaError_t gemm_bf16(const void* A, bool a_mn, int64_t a_row_bytes, const void* B, bool b_mn, int64_t b_row_bytes,
                      int64_t M, int32_t N, int32_t K, float* out, int64_t ldo, bool accumulate, cudaStream_t stream,
                      int num_sms);
// the two products of the f2 backward on that GEMM
cudaError_t tc_lmhead_grads(cudaStream_t stream, int num_sms, const void* weight, const void* hidden_chunk,
                            const void* D, int64_t ld, int64_t rows, int32_t d, int32_t V, float* dhidden_chunk,
                            float* dweight, bool beta_one);
cudaError_t launch_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                   const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                   const float* tok_ecoef, const float* tok_entropy, float* dhidden, float* dweight,
                                   bool accumulate, void* dlogits_ws, int64_t chunk_rows, cudaStream_t stream,
                                   int num_sms);
cudaError_t launch_loss_from_logp(int64_t n, const float* tok_logp, const float* tok_entropy, const float* tok_old,
                                  const float* tok_ref, const int32_t* tok_slot, const float* adv_slot,
                                  const float* tok_adv, const float* tok_weight, const double* n_global,
                                  const echo_loss_config& cfg, float* tok_loss, uint8_t* tok_flags, float* tok_coef,
                                  float* tok_ecoef, cudaStream_t stream, int num_sms);

size_t loss_stats_workspace_bytes();
cudaError_t launch_loss_stats(int64_t n, const float* tok_loss, const float* tok_logp, const float* tok_old,
                              const float* tok_ref, const float* tok_weight, const uint8_t* tok_flags, double* ws,
                              double* out, cudaStream_t stream);

}  // namespace echo
