// policy_loss.cu -- (3) streaming log-softmax + gather, (4) clipped surrogate + KL, (5) dL/dlogits in place.
//
// Per packed token t (one row of the [N x V] logits; PAPER.md :170 log pi_theta(a|s), :278 PPO/GRPO
// family, SPEC.md :219 objective):
//   pass 1  (m, s) = online max / sum-exp over the row, fp32 accumulation; z_a picked up on the way
//   scalar  lse = m + log s; logp = z_a - lse; rho, pg, kl, l_t, c_t  (echo::row_epilogue)
//   pass 2  logits[t, v] <- c_t (delta_{v,a} - exp(z_v - lse))  (bf16/fp32, RNE), in place
// The path is a memory-bound stream (no contraction): the design goal is exactly one HBM read and one HBM
// write per logit, 128-bit accesses, and nothing else on the memory bus.
//
// Kernels (one dispatch, echo_policy_loss_fwd_bwd_ex / _v2):
//   ECHO_ALGO_OCT_REG (AUTO) / QUAD_REG / QUAD_REG_EXACT (policy_loss_quad.cu; bf16, V <= 155648) -- the B200
//     design: an 8- (or 4-) CTA cluster owns a row, each CTA keeps its slice of the row in registers, 4 (or 2)
//     CTAs -- rows -- share an SM so that one row's MUFU-bound reduction overlaps the others' cluster merges and
//     store bursts; rows are handed out in order by a global counter and arrive through a TMA-fed shared-memory
//     ring; the CTA partials are merged through DSMEM (st.async + mbarrier); exactly one HBM read and one HBM
//     write per logit.
//   ECHO_ALGO_ROW_L2 (policy_loss_row.cu; bf16 or fp32, any V) -- one 1024-thread CTA per row, persistent over
//     rows; pass 1 loads with L2 evict_last, pass 2 re-loads (an L2 hit when the ~45 MB of rows in flight stay
//     resident) with evict_first and stores in place.  Generic path for fp32 and out-of-range vocabularies.
//
// Determinism: every row is reduced by the same thread layout (vector j of a row always belongs to the
// same thread, xor-butterfly warp merges, fixed warp order, rank-ordered cluster merge), so results
// depend only on (V, tile constants) -- not on the grid, the micro-batch split or the rank.
#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

// ====================================================================== dispatch
// How many clusters of `fn` can be resident at once (GPC shapes may strand SMs).  The persistent grids are sized
// to exactly that, so no cluster waits for a second wave.
int max_active_clusters(const void* fn, int threads, size_t smem, int cluster, int fallback) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 4096);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    return fallback;
  }
  return n;
}

cudaError_t launch_policy_loss(const LossParams& p, int32_t dtype, int algo, cudaStream_t stream, int num_sms,
                               LaunchShape* shape) {
  if (algo == ECHO_ALGO_QUAD_REG) return launch_quad(p, true, stream, num_sms, shape);
  if (algo == ECHO_ALGO_QUAD_REG_EXACT) return launch_quad(p, false, stream, num_sms, shape);
  if (algo == ECHO_ALGO_OCT_REG) return launch_oct(p, stream, num_sms, shape);
  if (algo == ECHO_ALGO_HEX_REG) return launch_hex(p, dtype, stream, num_sms, shape);
  return launch_row(p, dtype, stream, num_sms, shape);
}

}  // namespace echo
