// loss_logp.cu -- (4) from log-probs alone: the clipped surrogate, KL and entropy bonus of a token and its gradient
// coefficient c_t = dl_t/dlogp * grad_scale * w_t, for paths that produce logp without the logits (f2's fused LM head,
// f1).  Same scalar arithmetic as the fused kernels' row epilogue (echo::row_epilogue with lse = 0, z_a = logp), so a
// token gets the same loss, flags and coefficient whichever path computed its logp.
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

struct LogpLossParams {
  int64_t n;
  const float* __restrict__ tok_logp;
  const float* __restrict__ tok_entropy;
  const float* __restrict__ tok_old;
  const float* __restrict__ tok_ref;
  const int32_t* __restrict__ tok_slot;
  const float* __restrict__ adv_slot;
  const float* __restrict__ tok_adv;
  const float* __restrict__ tok_weight;
  const double* __restrict__ n_global;
  LossOpts o;
  float grad_scale;
  float* __restrict__ tok_loss;
  uint8_t* __restrict__ tok_flags;
  float* __restrict__ tok_coef;
  float* __restrict__ tok_ecoef;
};

__global__ void __launch_bounds__(256) loss_from_logp_kernel(const LogpLossParams p) {
  const float gscale = p.tok_weight ? p.grad_scale : (float)((double)p.grad_scale / *p.n_global);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.n; t += (int64_t)gridDim.x * blockDim.x) {
    const float adv = p.tok_adv ? p.tok_adv[t] : p.adv_slot[p.tok_slot[t]];
    const float ref = p.o.kl_coef > 0.0f ? p.tok_ref[t] : 0.0f;
    const float H = p.o.entropy_coef > 0.0f ? p.tok_entropy[t] : 0.0f;
    const float w = p.tok_weight ? p.tok_weight[t] : 1.0f;
    const RowScalars r = row_epilogue(0.0f, p.tok_logp[t], p.tok_old[t], ref, adv, p.o, gscale * w, H);
    p.tok_loss[t] = r.loss;
    p.tok_flags[t] = r.flags;
    p.tok_coef[t] = r.coef;
    if (p.tok_ecoef) p.tok_ecoef[t] = r.ecoef;
  }
}

cudaError_t launch_loss_from_logp(int64_t n, const float* tok_logp, const float* tok_entropy, const float* tok_old,
                                  const float* tok_ref, const int32_t* tok_slot, const float* adv_slot,
                                  const float* tok_adv, const float* tok_weight, const double* n_global,
                                  const echo_loss_config& cfg, float* tok_loss, uint8_t* tok_flags, float* tok_coef,
                                  float* tok_ecoef, cudaStream_t stream, int num_sms) {
  if (n == 0) return cudaSuccess;
  LogpLossParams p{n,        tok_logp, tok_entropy, tok_old, tok_ref, tok_slot, adv_slot, tok_adv, tok_weight,
                   n_global, LossOpts{cfg.clip_low, cfg.clip_high, cfg.clip_dual, cfg.kl_coef, cfg.kl_estimator,
                                      cfg.entropy_coef},
                   cfg.grad_scale, tok_loss, tok_flags, tok_coef, tok_ecoef};
  const int64_t blocks = (n + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 4 * num_sms ? blocks : 4 * num_sms);
  loss_from_logp_kernel<<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace echo
