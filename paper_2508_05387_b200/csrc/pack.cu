// pack.cu -- (1) version-lag filter + pack (PAPER.md :192, :201, :224; SPEC.md :44-49, :344).
//
// Three launches, integer work only (bit-exact):
//   pack_scan_kernel     1 CTA x 1024 threads: validate every rollout, decide keep per group from its
//                        version (keep iff t_train - v <= max_lag), exclusive-scan kept rollouts and
//                        their lengths into kept_rollout / kept_offset, min-reduce the error key.
//   pack_gather_kernel   grid-stride over kept slots: copy each kept rollout's first L tokens
//                        (action, old, ref) into the packed arrays, tag tok_slot, check action range.
//   pack_finalize_kernel 1 thread: decode the error key into status / first_bad_rollout.
// The error key is rollout * 8 + check (checks ordered FUTURE < MIXED < BAD_LENGTH < BAD_ACTION), so the
// reported error is the (rollout, check) lexicographic minimum -- independent of thread scheduling.
#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

constexpr int kScanThreads = 1024;
constexpr unsigned long long kNoError = 0xFFFFFFFFFFFFFFFFull;

__global__ void __launch_bounds__(kScanThreads) pack_scan_kernel(
    int32_t R, int32_t G, int32_t S, int64_t t_train, int32_t max_lag, int64_t rollout_base,
    const int64_t* __restrict__ version, const int32_t* __restrict__ resp_len, int32_t* __restrict__ kept_rollout,
    int64_t* __restrict__ kept_offset, echo_pack_result* __restrict__ res, int32_t filter_mode) {
  __shared__ unsigned long long s_err;
  __shared__ int32_t s_groups;  // filter_mode 1: groups with at least one kept rollout
  __shared__ int32_t s_wkeep[32];
  __shared__ int64_t s_wtok[32];
  __shared__ int32_t s_carry_keep;
  __shared__ int64_t s_carry_tok;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_err = kNoError;
    s_carry_keep = 0;
    s_carry_tok = 0;
    s_groups = 0;
  }
  __syncthreads();

  for (int32_t base = 0; base < R; base += kScanThreads) {
    const int32_t i = base + tid;
    int32_t keep = 0;
    int64_t len = 0;
    if (i < R) {
      const int64_t v = version[i];
      const int64_t v0 = version[(i / G) * G];
      const int32_t L = resp_len[i];
      unsigned long long key = kNoError;
      if (v > t_train)
        key = (unsigned long long)i * 8 + ECHO_DATA_FUTURE_VERSION;
      else if (filter_mode == 0 && v != v0)
        key = (unsigned long long)i * 8 + ECHO_DATA_MIXED_GROUP_VERSION;
      else if (L < 1 || L > S)
        key = (unsigned long long)i * 8 + ECHO_DATA_BAD_LENGTH;
      if (key != kNoError) atomicMin(&s_err, key);
      keep = (t_train - (filter_mode == 0 ? v0 : v)) <= (int64_t)max_lag ? 1 : 0;
      if (filter_mode == 1 && keep) {  // the group's first survivor counts the group
        bool first = true;
        for (int32_t j = (i / G) * G; j < i; ++j)
          if ((t_train - version[j]) <= (int64_t)max_lag) first = false;
        if (first) atomicAdd(&s_groups, 1);
      }
      len = keep ? (int64_t)min(max(L, 0), S) : 0;
    }
    // block-wide exclusive scan of (keep, len): warp inclusive scan, then warp totals
    int32_t ik = keep;
    int64_t it = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t k2 = __shfl_up_sync(0xffffffffu, ik, o);
      int64_t t2 = __shfl_up_sync(0xffffffffu, it, o);
      if (lane >= o) {
        ik += k2;
        it += t2;
      }
    }
    if (lane == 31) {
      s_wkeep[warp] = ik;
      s_wtok[warp] = it;
    }
    __syncthreads();
    if (warp == 0) {
      int32_t wk = s_wkeep[lane];
      int64_t wt = s_wtok[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t k2 = __shfl_up_sync(0xffffffffu, wk, o);
        int64_t t2 = __shfl_up_sync(0xffffffffu, wt, o);
        if (lane >= o) {
          wk += k2;
          wt += t2;
        }
      }
      s_wkeep[lane] = wk;  // inclusive over warps
      s_wtok[lane] = wt;
    }
    __syncthreads();
    const int32_t excl_k = s_carry_keep + (warp ? s_wkeep[warp - 1] : 0) + ik - keep;
    const int64_t excl_t = s_carry_tok + (warp ? s_wtok[warp - 1] : 0) + it - len;
    if (keep) {
      kept_rollout[excl_k] = (int32_t)(rollout_base + i);
      kept_offset[excl_k] = excl_t;
    }
    __syncthreads();
    if (tid == 0) {
      s_carry_keep += s_wkeep[31];
      s_carry_tok += s_wtok[31];
    }
    __syncthreads();
  }
  if (tid == 0) {
    kept_offset[s_carry_keep] = s_carry_tok;
    res->n_rollouts_kept = s_carry_keep;
    res->n_groups_kept = filter_mode == 0 ? s_carry_keep / G : s_groups;
    res->n_tokens = s_carry_tok;
    res->internal = (int64_t)s_err;
    res->status = ECHO_DATA_OK;
    res->first_bad_rollout = -1;
  }
}

__global__ void __launch_bounds__(256) pack_gather_kernel(
    int32_t S, int32_t V, int64_t rollout_base, int64_t cap, const int32_t* __restrict__ action,
    const float* __restrict__ old_logp, const float* __restrict__ ref_logp, const float* __restrict__ aux,
    const int32_t* __restrict__ kept_rollout, const int64_t* __restrict__ kept_offset, int32_t* __restrict__ tok_slot,
    int32_t* __restrict__ tok_action, float* __restrict__ tok_old, float* __restrict__ tok_ref,
    float* __restrict__ tok_aux, echo_pack_result* __restrict__ res) {
  __shared__ unsigned long long s_bad;
  const int32_t n_kept = res->n_rollouts_kept;
  const bool write = res->n_tokens <= cap;
  for (int32_t k = blockIdx.x; k < n_kept; k += gridDim.x) {
    if (threadIdx.x == 0) s_bad = kNoError;
    __syncthreads();
    const int64_t i = (int64_t)kept_rollout[k] - rollout_base;
    const int64_t off = kept_offset[k];
    const int32_t L = (int32_t)(kept_offset[k + 1] - off);
    const int64_t src = i * S;
    for (int32_t j = threadIdx.x; j < L; j += blockDim.x) {
      const int32_t a = action[src + j];
      if (a < 0 || a >= V) s_bad = (unsigned long long)i * 8 + ECHO_DATA_BAD_ACTION;  // same value from all
      if (write) {
        tok_slot[off + j] = k;
        tok_action[off + j] = a;
        tok_old[off + j] = old_logp[src + j];
        if (tok_ref) tok_ref[off + j] = ref_logp[src + j];
        if (tok_aux) tok_aux[off + j] = aux[src + j];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_bad != kNoError)
      atomicMin(reinterpret_cast<unsigned long long*>(&res->internal), s_bad);
  }
}

__global__ void pack_finalize_kernel(int64_t rollout_base, int64_t cap, echo_pack_result* res) {
  const unsigned long long key = (unsigned long long)res->internal;
  if (key != kNoError) {
    res->status = (int32_t)(key % 8);
    res->first_bad_rollout = (int32_t)(rollout_base + (int64_t)(key / 8));
  } else if (res->n_tokens > cap) {
    res->status = ECHO_DATA_CAPACITY;
    res->first_bad_rollout = -1;
  } else {
    res->status = ECHO_DATA_OK;
    res->first_bad_rollout = -1;
  }
}

cudaError_t launch_pack(int32_t R, int32_t G, int32_t S, int32_t V, int64_t t_train, int32_t max_lag,
                        int64_t rollout_base, const int64_t* version, const int32_t* resp_len, const int32_t* action,
                        const float* old_logp, const float* ref_logp, const float* aux, int64_t cap,
                        int32_t* kept_rollout, int64_t* kept_offset, int32_t* tok_slot, int32_t* tok_action,
                        float* tok_old, float* tok_ref, float* tok_aux, echo_pack_result* res, cudaStream_t stream,
                        int num_sms, int32_t filter_mode) {
  pack_scan_kernel<<<1, kScanThreads, 0, stream>>>(R, G, S, t_train, max_lag, rollout_base, version, resp_len,
                                                   kept_rollout, kept_offset, res, filter_mode);
  int grid = R < num_sms * 8 ? (R > 0 ? R : 1) : num_sms * 8;
  pack_gather_kernel<<<grid, 256, 0, stream>>>(S, V, rollout_base, cap, action, old_logp, ref_logp, aux,
                                               kept_rollout, kept_offset, tok_slot, tok_action, tok_old, tok_ref,
                                               tok_aux, res);
  pack_finalize_kernel<<<1, 1, 0, stream>>>(rollout_base, cap, res);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------------- f3
// Staleness histogram of a step (SPEC.md :373 version_histogram, :604 staleness_histogram): per rollout, lag =
// t_train - version, kept by its group's version as in pack_scan_kernel; counts of rollouts and tokens per lag bin
// for kept and dropped rollouts.  One CTA: shared-memory integer atomics (order-independent, bit-exact), then
// plain stores of every bin (hist needs no initialisation).
__global__ void __launch_bounds__(1024) staleness_hist_kernel(int32_t R, int32_t G, int32_t S, int64_t t_train,
                                                              int32_t max_lag, const int64_t* __restrict__ version,
                                                              const int32_t* __restrict__ resp_len, int32_t n_bins,
                                                              long long* __restrict__ hist, int32_t filter_mode) {
  extern __shared__ unsigned long long s_hist[];
  const int32_t nb = n_bins + 2;
  for (int32_t k = threadIdx.x; k < 4 * nb; k += blockDim.x) s_hist[k] = 0ull;
  __syncthreads();
  for (int32_t i = threadIdx.x; i < R; i += blockDim.x) {
    const int64_t lag = t_train - version[i];
    const bool kept = (t_train - version[filter_mode == 0 ? (i / G) * G : i]) <= (int64_t)max_lag;
    const int32_t bin = lag < 0 ? 0 : (lag < n_bins ? (int32_t)lag + 1 : n_bins + 1);
    const int32_t L = min(max(resp_len[i], 0), S);
    atomicAdd(&s_hist[(kept ? 0 : 1) * nb + bin], 1ull);
    atomicAdd(&s_hist[(kept ? 2 : 3) * nb + bin], (unsigned long long)L);
  }
  __syncthreads();
  for (int32_t k = threadIdx.x; k < 4 * nb; k += blockDim.x) hist[k] = (long long)s_hist[k];
}

cudaError_t launch_staleness_hist(int32_t R, int32_t G, int32_t S, int64_t t_train, int32_t max_lag,
                                  const int64_t* version, const int32_t* resp_len, int32_t n_bins, int64_t* hist,
                                  int32_t filter_mode, cudaStream_t stream) {
  const size_t smem = (size_t)4 * (n_bins + 2) * sizeof(unsigned long long);
  if (smem > 48 * 1024) {  // n_bins > 1534: past the default dynamic shared-memory limit (ABI allows 4096 bins)
    cudaError_t e = cudaFuncSetAttribute(staleness_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  staleness_hist_kernel<<<1, 1024, smem, stream>>>(R, G, S, t_train, max_lag, version, resp_len, n_bins,
                                                   reinterpret_cast<long long*>(hist), filter_mode);
  return cudaGetLastError();
}

}  // namespace echo
