// lmhead_bwd.cu -- f2 backward: dhidden = D W and dweight (+)= D^T h through the LM head, with
// D = dL/dz recomputed tile by tile on the tensor cores (lmhead_tile_kernel<.., 2>, this library's kernel) into a
// bf16 chunk buffer, and the two products as plain cuBLAS bf16 GEMMs (fp32 accumulation and output) on the caller's
// handle and stream.  Chunks of chunk_rows tokens bound the D buffer (chunk_rows x ld x 2 bytes).
#include <cublas_v2.h>

#include "echo_internal.h"

namespace echo {

cudaError_t launch_lmhead_backward(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                   const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                   const float* tok_ecoef, const float* tok_entropy, float* dhidden, float* dweight,
                                   bool accumulate, void* dlogits_ws, int64_t chunk_rows, void* cublas_handle,
                                   cudaStream_t stream, int num_sms, int* cublas_status) {
  *cublas_status = 0;
  cublasHandle_t h = static_cast<cublasHandle_t>(cublas_handle);
  const int64_t ld = ((int64_t)V + 7) & ~(int64_t)7;
  if (cublasSetStream(h, stream) != CUBLAS_STATUS_SUCCESS ||
      cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST) != CUBLAS_STATUS_SUCCESS) {
    *cublas_status = 1;
    return cudaErrorUnknown;
  }
  const float one = 1.0f, zero = 0.0f;
  const uint16_t* hid = static_cast<const uint16_t*>(hidden);
  for (int64_t r0 = 0; r0 < n_rows; r0 += chunk_rows) {
    const int64_t rows = (n_rows - r0 < chunk_rows) ? n_rows - r0 : chunk_rows;
    cudaError_t e = launch_lmhead_dlogits(hid + r0 * d, weight, rows, d, V, tok_action + r0, tok_lse + r0,
                                          tok_coef + r0, tok_ecoef ? tok_ecoef + r0 : nullptr,
                                          tok_ecoef ? tok_entropy + r0 : nullptr, dlogits_ws, ld, stream, num_sms);
    if (e != cudaSuccess) return e;
    // column-major view: dhidden^T (d x rows) = W^T (d x V) . D^T (V x rows)
    cublasStatus_t s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, d, (int)rows, V, &one, weight, CUDA_R_16BF, d,
                                    dlogits_ws, CUDA_R_16BF, (int)ld, &zero, dhidden + r0 * d, CUDA_R_32F, d,
                                    CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (s != CUBLAS_STATUS_SUCCESS) {
      *cublas_status = (int)s;
      return cudaErrorUnknown;
    }
    // dweight^T (d x V) (+)= h^T (d x rows) . D (rows x V)
    const float* beta = (accumulate || r0 > 0) ? &one : &zero;
    s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, d, V, (int)rows, &one, hid + r0 * d, CUDA_R_16BF, d, dlogits_ws,
                     CUDA_R_16BF, (int)ld, beta, dweight, CUDA_R_32F, d, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (s != CUBLAS_STATUS_SUCCESS) {
      *cublas_status = (int)s;
      return cudaErrorUnknown;
    }
  }
  return cudaGetLastError();
}

}  // namespace echo
