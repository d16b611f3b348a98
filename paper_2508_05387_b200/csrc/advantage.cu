// advantage.cu -- (2) GRPO group-relative advantage (PAPER.md :374; formula SPEC.md :209-213).
//
// One CTA of 256 threads over the kept rollouts in tiles of 256.  A group is the run of consecutive kept
// rollouts with the same kept_rollout / G: G members when pack keeps whole groups, its n_g <= G survivors with
// pack's per-rollout filter (f3 partial groups).  The thread at a run's first rollout evaluates the run in fp64
// with explicit round-to-nearest intrinsics (no FMA contraction), in index order:
//   mean = (sum r)/n_g, std = sqrt(sum (r-mean)^2 / n_g), A = (r-mean)/(std+eps) -> fp32 (RNE)
// so the result is bit-identical to a sequential IEEE evaluation.  The per-group statistics partials are
// folded by thread 0 in ascending order (fixed order => bitwise reproducible).  n_kept <= R is tiny (a few
// thousand): latency, not bandwidth, is all that matters.
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

constexpr int kAdvThreads = 256;

__global__ void __launch_bounds__(kAdvThreads) group_advantage_kernel(
    int32_t G, float eps, int64_t rollout_base, const float* __restrict__ reward,
    const int32_t* __restrict__ kept_rollout, const echo_pack_result* __restrict__ pack, float* __restrict__ adv_slot,
    double* __restrict__ adv_stats) {
  __shared__ double s_part[kAdvThreads][4];
  __shared__ double s_zero[kAdvThreads];
  const int32_t n_kept = pack->n_rollouts_kept;
  const double deps = (double)eps;
  double tot[4] = {0.0, 0.0, 0.0, 0.0};
  double n_zero = 0.0;
  for (int32_t k0 = 0; k0 < n_kept; k0 += kAdvThreads) {
    const int32_t k = k0 + threadIdx.x;
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    double zero = 0.0;
    const int32_t grp = k < n_kept ? kept_rollout[k] / G : -1;
    if (k < n_kept && (k == 0 || kept_rollout[k - 1] / G != grp)) {  // first rollout of its run
      int32_t k1 = k + 1;
      while (k1 < n_kept && kept_rollout[k1] / G == grp) ++k1;
      const double n_g = (double)(k1 - k);
      double sum = 0.0;
      for (int32_t j = k; j < k1; ++j) sum = __dadd_rn(sum, (double)reward[kept_rollout[j] - rollout_base]);
      const double mean = __ddiv_rn(sum, n_g);
      double ss = 0.0;
      for (int32_t j = k; j < k1; ++j) {
        const double d = __dsub_rn((double)reward[kept_rollout[j] - rollout_base], mean);
        ss = __dadd_rn(ss, __dmul_rn(d, d));
      }
      const double sd = __dsqrt_rn(__ddiv_rn(ss, n_g));
      zero = (sd == 0.0) ? 1.0 : 0.0;
      const double denom = __dadd_rn(sd, deps);
      for (int32_t j = k; j < k1; ++j) {
        const double r = (double)reward[kept_rollout[j] - rollout_base];
        const float a = __double2float_rn(__ddiv_rn(__dsub_rn(r, mean), denom));
        adv_slot[j] = a;
        const double ad = (double)a;
        part[0] = __dadd_rn(part[0], ad);
        part[1] = __dadd_rn(part[1], __dmul_rn(ad, ad));
        part[2] = __dadd_rn(part[2], r);
        part[3] = __dadd_rn(part[3], __dmul_rn(r, r));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) s_part[threadIdx.x][q] = part[q];
    s_zero[threadIdx.x] = zero;
    __syncthreads();
    if (threadIdx.x == 0) {  // runs in ascending order; other threads contributed exact zeros
      const int32_t m = min(kAdvThreads, n_kept - k0);
      for (int32_t j = 0; j < m; ++j) {
        if (j > 0 && kept_rollout[k0 + j - 1] / G == kept_rollout[k0 + j] / G) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) tot[q] = __dadd_rn(tot[q], s_part[j][q]);
        n_zero = __dadd_rn(n_zero, s_zero[j]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) adv_stats[q] = tot[q];
    adv_stats[4] = n_zero;
    adv_stats[5] = (double)n_kept;
  }
}

cudaError_t launch_group_advantage(int32_t G, float eps, int64_t rollout_base, const float* reward,
                                   const int32_t* kept_rollout, const echo_pack_result* pack, float* adv_slot,
                                   double* adv_stats, cudaStream_t stream) {
  group_advantage_kernel<<<1, kAdvThreads, 0, stream>>>(G, eps, rollout_base, reward, kept_rollout, pack, adv_slot,
                                                         adv_stats);
  return cudaGetLastError();
}

}  // namespace echo
