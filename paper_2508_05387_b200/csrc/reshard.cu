// reshard.cu -- f3: rebuild the packed CSR after token-balanced resharding.
//
// After the stale filter (PAPER.md :224) the ranks hold different numbers of kept tokens; parallel.py moves whole
// kept rollouts between ranks (NCCL all-to-all of the packed per-token and per-rollout arrays) so that every rank
// holds ~N_global / W tokens.  A receiving rank then has the rollouts' lengths and their tokens, rollout-major,
// and needs the CSR of (1) back: kept_offset = exclusive prefix sum of the lengths, tok_slot[t] = the rollout of
// token t.  Integer work, bit-exact.
//
//   csr_scan_kernel  1 CTA x 1024 threads: exclusive scan of the lengths (negative lengths count as 0)
//   csr_fill_kernel  one CTA per rollout (grid-stride): tok_slot[kept_offset[i] .. kept_offset[i+1]) = i
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

constexpr int kCsrThreads = 1024;

__global__ void __launch_bounds__(kCsrThreads) csr_scan_kernel(int32_t n, const int32_t* __restrict__ lengths,
                                                               int64_t* __restrict__ offsets) {
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < n; base += kCsrThreads) {
    const int32_t i = base + tid;
    const int64_t len = i < n ? (int64_t)max(lengths[i], 0) : 0;
    int64_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int64_t carry = s_carry;
    const int64_t excl = carry + (warp > 0 ? s_warp[warp - 1] : 0) + incl - len;
    if (i < n) offsets[i] = excl;
    __syncthreads();
    if (tid == kCsrThreads - 1) s_carry = excl + len;
    __syncthreads();
  }
  if (tid == 0) offsets[n] = s_carry;
}

__global__ void __launch_bounds__(256) csr_fill_kernel(int32_t n, const int64_t* __restrict__ offsets,
                                                       int32_t* __restrict__ tok_slot) {
  for (int32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t lo = offsets[i], hi = offsets[i + 1];
    for (int64_t t = lo + threadIdx.x; t < hi; t += blockDim.x) tok_slot[t] = i;
  }
}

cudaError_t launch_csr_from_lengths(int32_t n, const int32_t* lengths, int64_t* offsets, int32_t* tok_slot,
                                    cudaStream_t stream, int num_sms) {
  csr_scan_kernel<<<1, kCsrThreads, 0, stream>>>(n, lengths, offsets);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || n == 0 || tok_slot == nullptr) return e;
  const int grid = n < num_sms * 8 ? n : num_sms * 8;
  csr_fill_kernel<<<grid, 256, 0, stream>>>(n, offsets, tok_slot);
  return cudaGetLastError();
}

}  // namespace echo
