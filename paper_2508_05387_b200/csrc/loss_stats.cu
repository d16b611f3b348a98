// loss_stats.cu -- fixed-order fp64 reduction of the per-token outputs into the 10-entry stats vector.
//
//   loss_stats = {sum l, sum (logp-old), sum k3(ref,logp), n_clipped, n_nonfinite, rho_min, rho_max,
//                 sum logp, n_tokens, sum rho, sum w l}
// Launch 1: kStatBlocks (fixed) blocks; block b owns tokens [b*n/B, (b+1)*n/B) and reduces them with a
// fixed thread-strided loop + fixed shuffle tree into workspace[b].  Launch 2: one warp per statistic folds
// the B partials in a fixed order (contiguous lane ranges, then an xor tree).  The partition depends only on n_tokens, so the result is bitwise
// reproducible (and the W-rank all-reduce of these vectors only changes the order of B-level sums).
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

constexpr int kStatBlocks = 296;  // 2 x 148 SMs
constexpr int kStatThreads = 256;
constexpr int kNStat = 11;

struct Acc {
  double v[kNStat];
};

ECHO_DEVINL void acc_init(Acc& a) {
#pragma unroll
  for (int i = 0; i < kNStat; ++i) a.v[i] = 0.0;
  a.v[5] = INFINITY;
  a.v[6] = -INFINITY;
}
ECHO_DEVINL void acc_merge(Acc& a, const Acc& b) {
#pragma unroll
  for (int i = 0; i < kNStat; ++i) a.v[i] = (i == 5) ? fmin(a.v[i], b.v[i]) : (i == 6) ? fmax(a.v[i], b.v[i])
                                                                                          : a.v[i] + b.v[i];
}

__global__ void __launch_bounds__(kStatThreads) loss_stats_partial_kernel(
    int64_t n, const float* __restrict__ tok_loss, const float* __restrict__ tok_logp, const float* __restrict__ tok_old,
    const float* __restrict__ tok_ref, const float* __restrict__ tok_weight, const uint8_t* __restrict__ tok_flags,
    double* __restrict__ ws) {
  __shared__ double s[kStatThreads / 32][kNStat];
  const int64_t lo = (int64_t)blockIdx.x * n / kStatBlocks, hi = (int64_t)(blockIdx.x + 1) * n / kStatBlocks;
  Acc a;
  acc_init(a);
  for (int64_t t = lo + threadIdx.x; t < hi; t += kStatThreads) {
    const float logp = tok_logp[t], old = tok_old[t];
    const uint8_t f = tok_flags[t];
    a.v[0] += (double)tok_loss[t];
    a.v[1] += (double)logp - (double)old;
    if (tok_ref) {
      const double x = (double)tok_ref[t] - (double)logp;
      a.v[2] += exp(x) - x - 1.0;
    }
    a.v[3] += (double)(f & ECHO_FLAG_CLIPPED);
    a.v[4] += (double)((f & ECHO_FLAG_NONFINITE) ? 1 : 0);
    if (!(f & ECHO_FLAG_NONFINITE)) {
      const double rho = exp((double)logp - (double)old);
      a.v[5] = fmin(a.v[5], rho);
      a.v[6] = fmax(a.v[6], rho);
      a.v[9] += rho;
    }
    a.v[7] += (double)logp;
    a.v[8] += 1.0;
    a.v[10] += (tok_weight ? (double)tok_weight[t] : 1.0) * (double)tok_loss[t];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    Acc b;
#pragma unroll
    for (int i = 0; i < kNStat; ++i) b.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], o);
    acc_merge(a, b);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < kNStat; ++i) s[warp][i] = a.v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc tot;
#pragma unroll
    for (int i = 0; i < kNStat; ++i) tot.v[i] = s[0][i];
    for (int w = 1; w < kStatThreads / 32; ++w) {
      Acc b;
#pragma unroll
      for (int i = 0; i < kNStat; ++i) b.v[i] = s[w][i];
      acc_merge(tot, b);
    }
#pragma unroll
    for (int i = 0; i < kNStat; ++i) ws[blockIdx.x * kNStat + i] = tot.v[i];
  }
}

// One warp per statistic: lane l folds the partials [l B/32, (l+1) B/32) in order, then a fixed xor tree.
__global__ void __launch_bounds__(32 * kNStat) loss_stats_final_kernel(const double* __restrict__ ws,
                                                                      double* __restrict__ out) {
  const int i = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lo = lane * kStatBlocks / 32, hi = (lane + 1) * kStatBlocks / 32;
  double v = (i == 5) ? INFINITY : (i == 6) ? -INFINITY : 0.0;
  for (int b = lo; b < hi; ++b) {
    const double x = ws[b * kNStat + i];
    v = (i == 5) ? fmin(v, x) : (i == 6) ? fmax(v, x) : v + x;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = (i == 5) ? fmin(v, x) : (i == 6) ? fmax(v, x) : v + x;
  }
  if (lane == 0) out[i] = v;
}

size_t loss_stats_workspace_bytes() { return sizeof(double) * kStatBlocks * kNStat; }

cudaError_t launch_loss_stats(int64_t n, const float* tok_loss, const float* tok_logp, const float* tok_old,
                              const float* tok_ref, const float* tok_weight, const uint8_t* tok_flags, double* ws,
                              double* out, cudaStream_t stream) {
  loss_stats_partial_kernel<<<kStatBlocks, kStatThreads, 0, stream>>>(n, tok_loss, tok_logp, tok_old, tok_ref,
                                                                      tok_weight, tok_flags, ws);
  loss_stats_final_kernel<<<1, 32 * kNStat, 0, stream>>>(ws, out);
  return cudaGetLastError();
}

}  // namespace echo
