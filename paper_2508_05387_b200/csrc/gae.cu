// gae.cu -- f4: PPO-GAE per-token advantages from a trajectory's per-step rewards and values
// (the `rewards` and `values` fields of PAPER.md :163-164, "(s, a, log pi(a|s), v(s), r) ... required by PPO and
// its popular variants", :170-171).
//
// For each rollout i with length L_i, backwards from the last step (generalised advantage estimation):
//   delta_t = r_t + gamma V_{t+1} - V_t      (V_{L} = bootstrap_value[i], 0 when NULL / terminal)
//   A_t     = delta_t + gamma lambda A_{t+1}  (A_L = 0)
//   ret_t   = A_t + V_t
// One thread per rollout, fp64 with explicit round-to-nearest intrinsics in exactly this order (no FMA
// contraction), rounded to fp32 at the end: bit-identical to a sequential fp64 evaluation.  Positions >= L_i
// are not written.  The recursion is latency-bound and tiny (R <= a few thousand, L <= 8192).
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

__global__ void __launch_bounds__(128) gae_kernel(int32_t R, int32_t S, const int32_t* __restrict__ resp_len,
                                                  const float* __restrict__ rewards, const float* __restrict__ values,
                                                  const float* __restrict__ bootstrap, double gamma, double gl,
                                                  float* __restrict__ adv, float* __restrict__ ret) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R) return;
  const int32_t L = min(max(resp_len[i], 0), S);
  const int64_t base = (int64_t)i * S;
  double v_next = bootstrap ? (double)bootstrap[i] : 0.0;
  double a = 0.0;
  for (int32_t t = L - 1; t >= 0; --t) {
    const double v = (double)values[base + t];
    const double delta = __dsub_rn(__dadd_rn((double)rewards[base + t], __dmul_rn(gamma, v_next)), v);
    a = __dadd_rn(delta, __dmul_rn(gl, a));
    adv[base + t] = __double2float_rn(a);
    if (ret) ret[base + t] = __double2float_rn(__dadd_rn(a, v));
    v_next = v;
  }
}

cudaError_t launch_gae(int32_t R, int32_t S, const int32_t* resp_len, const float* rewards, const float* values,
                       const float* bootstrap, float gamma, float lam, float* adv, float* ret, cudaStream_t stream) {
  if (R == 0) return cudaSuccess;
  const double g = (double)gamma, gl = (double)gamma * (double)lam;  // exact: two fp32 significands fit in fp64
  gae_kernel<<<(R + 127) / 128, 128, 0, stream>>>(R, S, resp_len, rewards, values, bootstrap, g, gl, adv, ret);
  return cudaGetLastError();
}

}  // namespace echo
