// lmhead_bwd.cu -- f2 backward: dhidden = D W and dweight (+)= D^T h through the LM head, where
// D = dL/dz of a chunk of tokens is a bf16 [rows x ld] buffer produced by this library's kernels, and the two products
// run on this library's tcgen05 GEMM (gemm.cu) with fp32 accumulation and output.  Chunks of chunk_rows
// tokens bound the buffer (chunk_rows x ld x 2 bytes).  Two ways to get D:
//   launch_lmhead_backward  D recomputed from h and W on the tensor cores (lmhead_tile_kernel<.., 2>), given the
//                           forward's lse / entropy and echo_loss_from_logp's coefficients
//   (abi.cu) echo_lmhead_policy_loss_fwd_bwd  z = h W^T stored as bf16 (lmhead_tile_kernel<.., 3>), then the fused
//                           policy-loss kernel of (3)-(5) turns the chunk into D in place
#include "echo_internal.h"

namespace echo {

cudaError_t launch_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                   const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                   const float* tok_ecoef, const float* tok_entropy, float* dhidden, float* dweight,
                                   bool accumulate, void* dlogits_ws, int64_t chunk_rows, cudaStream_t stream,
                                   int num_sms) {
  const int64_t ld = ((int64_t)V + 7) & ~(int64_t)7;
  const uint16_t* hid = static_cast<const uint16_t*>(hidden);
  for (int64_t r0 = 0; r0 < n_rows; r0 += chunk_rows) {
    const int64_t rows = (n_rows - r0 < chunk_rows) ? n_rows - r0 : chunk_rows;
    cudaError_t e = launch_lmhead_dlogits(hid + r0 * d, weight, rows, d, V, tok_action + r0, tok_lse + r0,
                                          tok_coef + r0, tok_ecoef ? tok_ecoef + r0 : nullptr,
                                          tok_ecoef ? tok_entropy + r0 : nullptr, dlogits_ws, ld, stream, num_sms);
    if (e != cudaSuccess) return e;
    e = tc_lmhead_grads(stream, num_sms, weight, hid + r0 * d, dlogits_ws, ld, rows, d, V, dhidden + r0 * d, dweight,
                        accumulate || r0 > 0);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace echo
