// policy_loss_row.cu -- ECHO_ALGO_ROW_L2 (see policy_loss.cu for the overview).
#include <cuda_bf16.h>

#include <atomic>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

// ====================================================================== ECHO_ALGO_ROW_L2
// Rows are handed out in order by a global counter (one {next row, CTAs done} pair per launch slot, reset by the
// launch's last CTA), so the CTAs work on one compact window of consecutive rows (see policy_loss_quad.cu).
constexpr int kRowSchedSlots = 256;
__device__ unsigned long long g_rowk_sched[kRowSchedSlots][2];

constexpr int kRThreads = 1024;
constexpr int kRWarps = kRThreads / 32;
constexpr int kRUnroll = 4;

template <int DT>  // 0 = fp32, 1 = bf16
struct RowVec;
template <>
struct RowVec<1> {
  static constexpr int N = 8;
  static ECHO_DEVINL void unpack(const uint4& w, float (&x)[8]) { unpack8(w, x); }
  static ECHO_DEVINL uint4 pack(const float (&x)[8]) {
    return make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                      pack_bf16x2(x[6], x[7]));
  }
  static ECHO_DEVINL float load1(const uint8_t* row, int32_t v) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(row)[v]);
  }
  static ECHO_DEVINL void store1(uint8_t* row, int32_t v, float x) {
    reinterpret_cast<__nv_bfloat16*>(row)[v] = __float2bfloat16_rn(x);
  }
};
template <>
struct RowVec<0> {
  static constexpr int N = 4;
  static ECHO_DEVINL void unpack(const uint4& w, float (&x)[4]) {
    x[0] = __uint_as_float(w.x); x[1] = __uint_as_float(w.y);
    x[2] = __uint_as_float(w.z); x[3] = __uint_as_float(w.w);
  }
  static ECHO_DEVINL uint4 pack(const float (&x)[4]) {
    return make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
  }
  static ECHO_DEVINL float load1(const uint8_t* row, int32_t v) { return reinterpret_cast<const float*>(row)[v]; }
  static ECHO_DEVINL void store1(uint8_t* row, int32_t v, float x) { reinterpret_cast<float*>(row)[v] = x; }
};

// kGrad = false: forward-only log-probs, logits not written; kEnt: the f4 entropy bonus
template <int DT, bool kGrad, bool kEnt = false>
__global__ void __launch_bounds__(kRThreads, 1) policy_loss_row_kernel(const LossParams p) {
  using RV = RowVec<DT>;
  constexpr int N = RV::N;
  __shared__ float s_m[kRWarps], s_s[kRWarps], s_t[kRWarps];
  __shared__ float s_za, s_coef, s_lse_l2e, s_lse, s_H, s_ecoef;
  __shared__ long long s_row;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t V = p.V;
  const int32_t nvec = V / N;
  const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
  const float gscale = kGrad ? base_scale(p) : 0.0f;

  unsigned long long* const sched = g_rowk_sched[p.sched_slot];
  if (tid == 0) s_row = (long long)atomicAdd(&sched[0], 1ull);
  __syncthreads();
  for (int64_t row = s_row; row < p.n_rows; row = s_row) {
    // the next row is grabbed now and published at the end-of-row barrier (its latency stays off the path)
    unsigned long long next = 0;
    if (tid == 0) next = atomicAdd(&sched[0], 1ull);
    uint8_t* rowp = p.logits + row * p.ld_bytes;
    const int32_t a = p.tok_action[row];
    RowMeta meta{0.f, 0.f, 0.f};
    if (tid == 0) {
      meta = load_meta(p, row);
      s_za = NAN;
    }
    __syncthreads();

    // ---- pass 1
    MaxSum acc{-INFINITY, 0.0f};
    float tacc = 0.0f;
    for (int32_t v0 = tid; v0 < nvec; v0 += kRThreads * kRUnroll) {
      uint4 w[kRUnroll];
#pragma unroll
      for (int u = 0; u < kRUnroll; ++u) {
        const int32_t v = v0 + u * kRThreads;
        if (v < nvec) w[u] = ldg_v4_hint(rowp + (int64_t)v * 16, pol_keep);
      }
#pragma unroll
      for (int u = 0; u < kRUnroll; ++u) {
        const int32_t v = v0 + u * kRThreads;
        if (v < nvec) {
          float x[N];
          RV::unpack(w[u], x);
          const int32_t col = v * N;
          if ((uint32_t)(a - col) < (uint32_t)N) {
#pragma unroll
            for (int e = 0; e < N; ++e)
              if (col + e == a) s_za = x[e];
          }
          if (kEnt) online_update3<N>(acc, tacc, x);
          else online_update<N>(acc, x);
        }
      }
    }
    for (int32_t col = nvec * N + tid; col < V; col += kRThreads) {  // ragged tail (V % N)
      float x[1] = {RV::load1(rowp, col)};
      if (col == a) s_za = x[0];
      if (kEnt) online_update3<1>(acc, tacc, x);
      else online_update<1>(acc, x);
    }
    if (kEnt) {
      const MaxSum3 a3 = warp_maxsum3(acc.m, acc.s, tacc);
      acc = a3.ms;
      tacc = a3.t;
    } else {
      acc = warp_maxsum(acc);
    }
    if (lane == 0) {
      s_m[warp] = acc.m;
      s_s[warp] = acc.s;
      if (kEnt) s_t[warp] = tacc;
    }
    __syncthreads();
    MaxSum3 tot{MaxSum{-INFINITY, 0.0f}, 0.0f};
    if (warp == 0) {  // kRWarps == 32: one lane per warp
      if (kEnt) tot = warp_maxsum3(s_m[lane], s_s[lane], s_t[lane]);
      else tot.ms = warp_maxsum(MaxSum{s_m[lane], s_s[lane]});
    }
    if (tid == 0) {
      const float lse = tot.ms.m + logf(tot.ms.s);
      const float za = (a < 0 || a >= V) ? NAN : s_za;
      if constexpr (kGrad) {
        const float H = kEnt ? lse - tot.t / tot.ms.s : 0.0f;
        const RowScalars r = row_epilogue(lse, za, meta.old, meta.ref, meta.adv, loss_opts(p), gscale * meta.w, H);
        p.tok_logp[row] = r.logp;
        p.tok_loss[row] = r.loss;
        p.tok_flags[row] = r.flags;
        if (kEnt && p.tok_entropy) p.tok_entropy[row] = H;
        s_coef = r.coef;
        s_lse_l2e = lse * kLog2e;
        s_lse = lse;
        s_H = H;
        s_ecoef = r.ecoef;
      } else {
        const float logp = za - lse;
        p.tok_logp[row] = logp;
        if (p.tok_lse) p.tok_lse[row] = lse;
        if (p.tok_flags) p.tok_flags[row] = (isfinite(lse) && isfinite(logp)) ? 0 : ECHO_FLAG_NONFINITE;
      }
    }
    if (tid == 0) s_row = (long long)next;  // read by the loop condition after the barriers below
    __syncthreads();
    if constexpr (!kGrad) continue;
    const float coef = s_coef, lse_l2e = s_lse_l2e, lse = s_lse, H = s_H, ecoef = s_ecoef;

    // ---- pass 2
    for (int32_t v0 = tid; v0 < nvec; v0 += kRThreads * kRUnroll) {
      uint4 w[kRUnroll];
#pragma unroll
      for (int u = 0; u < kRUnroll; ++u) {
        const int32_t v = v0 + u * kRThreads;
        if (v < nvec) w[u] = ldg_v4_hint(rowp + (int64_t)v * 16, pol_drop);
      }
#pragma unroll
      for (int u = 0; u < kRUnroll; ++u) {
        const int32_t v = v0 + u * kRThreads;
        if (v < nvec) {
          float x[N];
          RV::unpack(w[u], x);
          if (kEnt) grad_values_ent<N>(x, v * N, a, coef, lse_l2e, lse, H, ecoef);
          else grad_values<N>(x, v * N, a, coef, lse_l2e);
          stg_v4_hint(rowp + (int64_t)v * 16, RV::pack(x), pol_drop);
        }
      }
    }
    for (int32_t col = nvec * N + tid; col < V; col += kRThreads) {
      float x[1] = {RV::load1(rowp, col)};
      if (kEnt) grad_values_ent<1>(x, col, a, coef, lse_l2e, lse, H, ecoef);
      else grad_values<1>(x, col, a, coef, lse_l2e);
      RV::store1(rowp, col, x[0]);
    }
    __syncthreads();  // s_* reuse by the next row
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&sched[1], 1ull) == (unsigned long long)gridDim.x - 1ull) {
      sched[0] = 0ull;
      sched[1] = 0ull;
    }
  }
}

cudaError_t launch_row(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms, LaunchShape* shape,
                       bool grad) {
  int64_t grid = num_sms;
  if (grid > p.n_rows) grid = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)grid, 1, kRThreads, 0};
    return cudaSuccess;
  }
  static std::atomic<uint32_t> next_slot{0}, next_slot_graph{0};
  LossParams q = p;
  q.sched_slot = (int32_t)next_sched_slot(next_slot, next_slot_graph, stream, kRowSchedSlots);
  const bool ent = grad && (p.entropy_coef > 0.0f || p.tok_entropy != nullptr);
  if (dtype == ECHO_BF16) {
    if (ent)
      policy_loss_row_kernel<1, true, true><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
    else if (grad)
      policy_loss_row_kernel<1, true><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
    else
      policy_loss_row_kernel<1, false><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
  } else {
    if (ent)
      policy_loss_row_kernel<0, true, true><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
    else if (grad)
      policy_loss_row_kernel<0, true><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
    else
      policy_loss_row_kernel<0, false><<<(unsigned)grid, kRThreads, 0, stream>>>(q);
  }
  return cudaGetLastError();
}

}  // namespace echo
