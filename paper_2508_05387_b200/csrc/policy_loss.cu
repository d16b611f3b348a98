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
// Two kernels:
//   ECHO_ALGO_CLUSTER_SMEM (policy_loss_cluster_kernel; bf16, V <= 196608) -- the B200 design.
//     A thread-block cluster of 2 CTAs (2 SMs) owns one row; each CTA owns half of it.  A producer warp
//     streams the half-row into a 26 x 8 KB shared-memory ring with 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx, L2 evict_first).  16 consumer warps run pass 1 straight out
//     of shared memory, reduce (m, s) warp -> CTA, and swap the CTA pair's partials through DSMEM with one
//     st.async that completes on the peer's mbarrier (no cluster-wide barrier per row, so the producer
//     never stalls).  Both CTAs merge the two partials in rank order -> identical lse bits.  Pass 2 reads
//     the half-row again from shared memory (not HBM), writes 16-byte gradient vectors, and frees ring
//     slots, which the producer immediately refills with the next row.  HBM traffic = 1R + 1W exactly,
//     independent of L2 behaviour; persistent grid of 74 clusters (148 SMs).
//   ECHO_ALGO_ROW_L2 (policy_loss_row_kernel; bf16 or fp32, any V) -- one 1024-thread CTA per row,
//     persistent over rows; pass 1 loads with L2 evict_last, pass 2 re-loads (an L2 hit when the ~45 MB
//     of rows in flight stay resident) with evict_first and stores in place.
//
// Determinism: every row is reduced by the same thread layout (vector j of a row always belongs to the
// same thread, xor-butterfly warp merges, fixed warp order, rank-0-then-rank-1 pair merge), so results
// depend only on (V, tile constants) -- not on the grid, the micro-batch split or the rank.
#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

// ====================================================================== shared per-row helpers
struct RowMeta {
  float old, ref, adv;
};
ECHO_DEVINL RowMeta load_meta(const LossParams& p, int64_t row) {
  RowMeta m;
  m.old = p.tok_old[row];
  m.ref = (p.kl_coef > 0.0f) ? p.tok_ref[row] : 0.0f;
  m.adv = p.adv_slot[p.tok_slot[row]];
  return m;
}

// Online update of (m, s) with N values already in registers.  -inf entries contribute 0.
template <int N>
ECHO_DEVINL void online_update(MaxSum& acc, const float (&x)[N]) {
  float cm = x[0];
#pragma unroll
  for (int e = 1; e < N; ++e) cm = fmaxf(cm, x[e]);
  if (cm > acc.m) {
    acc.s = acc.s * ex2((acc.m - cm) * kLog2e);
    acc.m = cm;
  }
  const float mb = (acc.m == -INFINITY) ? 0.0f : acc.m * kLog2e;
  float t = 0.0f;
#pragma unroll
  for (int e = 0; e < N; ++e) t += ex2(fmaf(x[e], kLog2e, -mb));
  acc.s += t;
}

ECHO_DEVINL void unpack8(const uint4& w, float (&x)[8]) {
  x[0] = bf16lo(w.x); x[1] = bf16hi(w.x);
  x[2] = bf16lo(w.y); x[3] = bf16hi(w.y);
  x[4] = bf16lo(w.z); x[5] = bf16hi(w.z);
  x[6] = bf16lo(w.w); x[7] = bf16hi(w.w);
}

// Gradient of N values: d_v = c (delta_{v,a} - p_v), p_v = 2^(z log2e - lse log2e).
template <int N>
ECHO_DEVINL void grad_values(float (&x)[N], int32_t col0, int32_t a, float coef, float lse_l2e) {
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float p = ex2(fmaf(x[e], kLog2e, -lse_l2e));
    x[e] = (col0 + e == a) ? fmaf(-coef, p, coef) : -coef * p;
  }
}

// ====================================================================== ECHO_ALGO_CLUSTER_SMEM
constexpr int kCConsumerWarps = 16;
constexpr int kCConsumers = kCConsumerWarps * 32;     // 512
constexpr int kCThreads = kCConsumers + 32;           // + 1 producer warp
constexpr int kCChunk = kCConsumers * 16;             // 8 KB: one 16-byte vector per consumer thread
constexpr int kCChunkElems = kCChunk / 2;             // 4096 bf16
constexpr int kCRing = 26;                            // 208 KB ring
constexpr int kCMaxChunksPerRow = 24;                 // leave >= 2 slots of prefetch head-room
constexpr int kCBarConsumers = 1;                     // named barrier id

struct __align__(128) ClusterSmem {
  uint8_t ring[kCRing][kCChunk];
  uint64_t full[kCRing];
  uint64_t empty[kCRing];
  uint64_t xbar[2];
  uint4 xbuf[2];  // peer's {m, s, z_a, -} for row parity 0 / 1
  float red_m[kCConsumerWarps];
  float red_s[kCConsumerWarps];
  float za;
  float coef;
  float lse_l2e;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCThreads, 1)
    policy_loss_cluster_kernel(const LossParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ClusterSmem& sm = *reinterpret_cast<ClusterSmem*>(smem_raw);
  const uint32_t rank = cluster_ctarank();
  const uint32_t cid = cluster_id_x(), ncl = nclusters_x();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int32_t V = p.V;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;  // rank 0: [0, h), rank 1: [h, V)
  const int32_t c0 = rank ? min(h, V) : 0;
  const int32_t c1 = rank ? V : min(h, V);
  const int32_t c1r = (c1 + 7) & ~7;
  const uint32_t slice_bytes = (uint32_t)(c1r - c0) * 2u;
  const int nchunks = (int)((slice_bytes + kCChunk - 1) / kCChunk);

  if (tid == 0) {
    for (int i = 0; i < kCRing; ++i) {
      mbar_init(smem_u32(&sm.full[i]), 1);
      mbar_init(smem_u32(&sm.empty[i]), kCConsumerWarps);
    }
    mbar_init(smem_u32(&sm.xbar[0]), 1);
    mbar_init(smem_u32(&sm.xbar[1]), 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();

  if (warp == kCConsumerWarps) {
    // ------------------------------------------------------------ producer: TMA bulk loads into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t q = 0;
      for (int64_t row = cid; row < p.n_rows; row += ncl) {
        const uint8_t* src = p.logits + row * p.ld_bytes + (int64_t)c0 * 2;
        for (int c = 0; c < nchunks; ++c, ++q) {
          const uint32_t slot = q % kCRing, round = q / kCRing;
          mbar_wait(smem_u32(&sm.empty[slot]), (round & 1) ^ 1);
          const uint32_t nb = min((uint32_t)kCChunk, slice_bytes - (uint32_t)c * kCChunk);
          mbar_arrive_expect_tx(smem_u32(&sm.full[slot]), nb);
          bulk_g2s(smem_u32(&sm.ring[slot][0]), src + (int64_t)c * kCChunk, nb, smem_u32(&sm.full[slot]), pol);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ consumers
    const uint32_t peer = rank ^ 1u;
    const uint32_t xbuf_remote0 = mapa(smem_u32(&sm.xbuf[0]), peer);
    const uint32_t xbar_remote0 = mapa(smem_u32(&sm.xbar[0]), peer);
    const uint64_t st_pol = policy_evict_first();
    const double n_global = *p.n_global;
    uint32_t q = 0, it = 0;
    for (int64_t row = cid; row < p.n_rows; row += ncl, ++it) {
      const int32_t a = p.tok_action[row];
      RowMeta meta{0.f, 0.f, 0.f};
      if (tid == 0) meta = load_meta(p, row);

      // ---- pass 1: online (max, sum-exp) over this CTA's half-row, straight from shared memory
      MaxSum acc{-INFINITY, 0.0f};
      const uint32_t q0 = q;
      for (int c = 0; c < nchunks; ++c, ++q) {
        const uint32_t slot = q % kCRing, round = q / kCRing;
        mbar_wait(smem_u32(&sm.full[slot]), round & 1);
        const int32_t col = c0 + c * kCChunkElems + tid * 8;
        if (col < c1) {
          float x[8];
          unpack8(lds_v4(smem_u32(&sm.ring[slot][tid * 16])), x);
          if (col + 8 > c1) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (col + e >= c1) x[e] = -INFINITY;
          }
          if ((uint32_t)(a - col) < 8u) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (col + e == a) sm.za = x[e];
          }
          online_update<8>(acc, x);
        }
      }
      acc = warp_maxsum(acc);
      if (lane == 0) {
        sm.red_m[warp] = acc.m;
        sm.red_s[warp] = acc.s;
      }
      named_bar_sync(kCBarConsumers, kCConsumers);

      // ---- CTA-pair merge through DSMEM + the scalar epilogue (thread 0 of each CTA)
      if (tid == 0) {
        MaxSum mine{sm.red_m[0], sm.red_s[0]};
        for (int w = 1; w < kCConsumerWarps; ++w) mine = maxsum_merge(mine, MaxSum{sm.red_m[w], sm.red_s[w]});
        const uint32_t par = it & 1u;
        const bool owner = (a >= c0 && a < c1);
        const float za_mine = owner ? sm.za : 0.0f;
        const uint32_t xbar_local = smem_u32(&sm.xbar[par]);
        mbar_arrive_expect_tx(xbar_local, 16);
        st_async_v4(xbuf_remote0 + par * 16u,
                    make_uint4(__float_as_uint(mine.m), __float_as_uint(mine.s), __float_as_uint(za_mine), 0u),
                    xbar_remote0 + par * 8u);
        mbar_wait_cluster(xbar_local, (it >> 1) & 1u);
        const uint4 msg = sm.xbuf[par];
        const MaxSum theirs{__uint_as_float(msg.x), __uint_as_float(msg.y)};
        const MaxSum tot = rank == 0 ? maxsum_merge(mine, theirs) : maxsum_merge(theirs, mine);
        const float lse = tot.m + logf(tot.s);
        float za = owner ? za_mine : __uint_as_float(msg.z);
        if (a < 0 || a >= V) za = NAN;
        const RowScalars r = row_epilogue(lse, za, meta.old, meta.ref, meta.adv, p.clip_low, p.clip_high,
                                          p.kl_coef, p.grad_scale, n_global);
        if (rank == 0) {
          p.tok_logp[row] = r.logp;
          p.tok_loss[row] = r.loss;
          p.tok_flags[row] = r.flags;
        }
        sm.coef = r.coef;
        sm.lse_l2e = lse * kLog2e;
      }
      named_bar_sync(kCBarConsumers, kCConsumers);
      const float coef = sm.coef, lse_l2e = sm.lse_l2e;

      // ---- pass 2: gradient from shared memory, 16-byte stores in place, free the ring slots
      uint8_t* dst_row = p.logits + row * p.ld_bytes;
      for (int c = 0; c < nchunks; ++c) {
        const uint32_t slot = (q0 + c) % kCRing;
        const int32_t col = c0 + c * kCChunkElems + tid * 8;
        if (col < c1) {
          float x[8];
          unpack8(lds_v4(smem_u32(&sm.ring[slot][tid * 16])), x);
          grad_values<8>(x, col, a, coef, lse_l2e);
          if (col + 8 <= c1) {
            const uint4 o = make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                                       pack_bf16x2(x[6], x[7]));
            stg_v4_hint(dst_row + (int64_t)col * 2, o, st_pol);
          } else {
            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dst_row) + col;
            for (int e = 0; e < 8 && col + e < c1; ++e) d[e] = __float2bfloat16_rn(x[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sm.empty[slot]));
      }
    }
  }
  cluster_sync_all();
}

// ====================================================================== ECHO_ALGO_ROW_L2
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

template <int DT>
__global__ void __launch_bounds__(kRThreads, 1) policy_loss_row_kernel(const LossParams p) {
  using RV = RowVec<DT>;
  constexpr int N = RV::N;
  __shared__ float s_m[kRWarps], s_s[kRWarps];
  __shared__ float s_za, s_coef, s_lse_l2e;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t V = p.V;
  const int32_t nvec = V / N;
  const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
  const double n_global = *p.n_global;

  for (int64_t row = blockIdx.x; row < p.n_rows; row += gridDim.x) {
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
          online_update<N>(acc, x);
        }
      }
    }
    for (int32_t col = nvec * N + tid; col < V; col += kRThreads) {  // ragged tail (V % N)
      float x[1] = {RV::load1(rowp, col)};
      if (col == a) s_za = x[0];
      online_update<1>(acc, x);
    }
    acc = warp_maxsum(acc);
    if (lane == 0) {
      s_m[warp] = acc.m;
      s_s[warp] = acc.s;
    }
    __syncthreads();
    if (tid == 0) {
      MaxSum tot{s_m[0], s_s[0]};
      for (int w = 1; w < kRWarps; ++w) tot = maxsum_merge(tot, MaxSum{s_m[w], s_s[w]});
      const float lse = tot.m + logf(tot.s);
      const float za = (a < 0 || a >= V) ? NAN : s_za;
      const RowScalars r = row_epilogue(lse, za, meta.old, meta.ref, meta.adv, p.clip_low, p.clip_high, p.kl_coef,
                                        p.grad_scale, n_global);
      p.tok_logp[row] = r.logp;
      p.tok_loss[row] = r.loss;
      p.tok_flags[row] = r.flags;
      s_coef = r.coef;
      s_lse_l2e = lse * kLog2e;
    }
    __syncthreads();
    const float coef = s_coef, lse_l2e = s_lse_l2e;

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
          grad_values<N>(x, v * N, a, coef, lse_l2e);
          stg_v4_hint(rowp + (int64_t)v * 16, RV::pack(x), pol_drop);
        }
      }
    }
    for (int32_t col = nvec * N + tid; col < V; col += kRThreads) {
      float x[1] = {RV::load1(rowp, col)};
      grad_values<1>(x, col, a, coef, lse_l2e);
      RV::store1(rowp, col, x[0]);
    }
    __syncthreads();  // s_* reuse by the next row
  }
}

// ====================================================================== launchers
bool cluster_algo_supports(int32_t dtype, int32_t V) {
  if (dtype != ECHO_BF16) return false;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;
  const int64_t bytes = (int64_t)h * 2;
  return V >= 2 * 8 && (bytes + kCChunk - 1) / kCChunk <= kCMaxChunksPerRow;
}

cudaError_t launch_policy_loss(const LossParams& p, int32_t dtype, int algo, cudaStream_t stream, int num_sms) {
  if (algo == ECHO_ALGO_CLUSTER_SMEM) {
    const size_t smem = sizeof(ClusterSmem);
    cudaError_t e = cudaFuncSetAttribute(policy_loss_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int64_t clusters = num_sms / 2;
    if (clusters > p.n_rows) clusters = p.n_rows;
    policy_loss_cluster_kernel<<<(unsigned)(clusters * 2), kCThreads, smem, stream>>>(p);
    return cudaGetLastError();
  }
  int64_t grid = num_sms;
  if (grid > p.n_rows) grid = p.n_rows;
  if (dtype == ECHO_BF16)
    policy_loss_row_kernel<1><<<(unsigned)grid, kRThreads, 0, stream>>>(p);
  else
    policy_loss_row_kernel<0><<<(unsigned)grid, kRThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace echo
