// lmhead_bwd.cu -- f2 backward: dhidden = D W and dweight (+)= D^T h through the LM head, where
// D = dL/dz of a chunk of tokens is a bf16 [rows x ld] buffer produced by this library's kernels, and the two products
// run on this library's tcgen05 GEMM (gemm.cu; cublas_handle NULL) or as cuBLAS bf16 GEMMs on the caller's handle
// and stream, both with fp32 accumulation and output.  Chunks of chunk_rows
// tokens bound the buffer (chunk_rows x ld x 2 bytes).  Two ways to get D:
//   launch_lmhead_backward  D recomputed from h and W on the tensor cores (lmhead_tile_kernel<.., 2>), given the
//                           forward's lse / entropy and echo_loss_from_logp's coefficients
//   (abi.cu) echo_lmhead_policy_loss_fwd_bwd  z = h W^T stored as bf16 (lmhead_tile_kernel<.., 3>), then the fused
//                           policy-loss kernel of (3)-(5) turns the chunk into D in place
#include <cublas_v2.h>

#include "echo_internal.h"

namespace echo {

int cublas_lmhead_grads(void* cublas_handle, cudaStream_t stream, const void* weight, const void* hidden_chunk,
                        const void* D, int64_t ld, int64_t rows, int32_t d, int32_t V, float* dhidden_chunk,
                        float* dweight, bool beta_one) {
  cublasHandle_t h = static_cast<cublasHandle_t>(cublas_handle);
  cublasStatus_t s = cublasSetStream(h, stream);
  if (s == CUBLAS_STATUS_SUCCESS) s = cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST);
  if (s != CUBLAS_STATUS_SUCCESS) return (int)s;
  const float one = 1.0f, zero = 0.0f;
  // column-major view: dhidden^T (d x rows) = W^T (d x V) . D^T (V x rows)
  s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, d, (int)rows, V, &one, weight, CUDA_R_16BF, d, D, CUDA_R_16BF,
                   (int)ld, &zero, dhidden_chunk, CUDA_R_32F, d, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (s != CUBLAS_STATUS_SUCCESS) return (int)s;
  // dweight^T (d x V) (+)= h^T (d x rows) . D (rows x V)
  s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, d, V, (int)rows, &one, hidden_chunk, CUDA_R_16BF, d, D, CUDA_R_16BF,
                   (int)ld, beta_one ? &one : &zero, dweight, CUDA_R_32F, d, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  return (int)s;
}

cudaError_t launch_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                   const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                   const float* tok_ecoef, const float* tok_entropy, float* dhidden, float* dweight,
                                   bool accumulate, void* dlogits_ws, int64_t chunk_rows, void* cublas_handle,
                                   cudaStream_t stream, int num_sms, int* cublas_status) {
  *cublas_status = 0;
  const int64_t ld = ((int64_t)V + 7) & ~(int64_t)7;
  const uint16_t* hid = static_cast<const uint16_t*>(hidden);
  for (int64_t r0 = 0; r0 < n_rows; r0 += chunk_rows) {
    const int64_t rows = (n_rows - r0 < chunk_rows) ? n_rows - r0 : chunk_rows;
    cudaError_t e = launch_lmhead_dlogits(hid + r0 * d, weight, rows, d, V, tok_action + r0, tok_lse + r0,
                                          tok_coef + r0, tok_ecoef ? tok_ecoef + r0 : nullptr,
                                          tok_ecoef ? tok_entropy + r0 : nullptr, dlogits_ws, ld, stream, num_sms);
    if (e != cudaSuccess) return e;
    if (!cublas_handle) {
      e = tc_lmhead_grads(stream, num_sms, weight, hid + r0 * d, dlogits_ws, ld, rows, d, V, dhidden + r0 * d, dweight,
                          accumulate || r0 > 0);
      if (e != cudaSuccess) return e;
      continue;
    }
    *cublas_status = cublas_lmhead_grads(cublas_handle, stream, weight, hid + r0 * d, dlogits_ws, ld, rows, d, V,
                                         dhidden + r0 * d, dweight, accumulate || r0 > 0);
    if (*cublas_status != 0) return cudaErrorUnknown;
  }
  return cudaGetLastError();
}

}  // namespace echo
