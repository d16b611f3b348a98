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

// ====================================================================== ECHO_ALGO_CLUSTER_REG
// Same CTA-pair / TMA-ring / DSMEM structure as CLUSTER_SMEM, but each consumer thread keeps its slice of the
// half-row in REGISTERS (kRegChunks x 16 B = 80 registers for Qwen's vocab), so a ring slot is released as
// soon as it has been copied into registers.  The 208 KB ring then only stages loads: while the consumers
// reduce and write back row k, the producer is already streaming row k+1 (and part of k+2) -> HBM never
// waits on the reduction.  Per row and thread:
//   pass 1a  copy chunk c from the ring into v[c] (free the slot), running max of its 8 values
//   pass 1b  e = 2^((z - m_t) log2e), s_t += e, and (kStoreExp) overwrite v[c] with e as packed fp16
//   merge    (m_t, s_t) -> warp -> CTA -> CTA pair (st.async) -> lse; epilogue -> c_t
//   pass 2   d = -c_t 2^((m_t - lse) log2e) e   (kStoreExp: one FMUL per logit, no MUFU)
//            d = -c_t 2^((z - lse) log2e)         (!kStoreExp: recompute from the bf16 logits)
//            the action column gets c_t (1 - p_a) from the fp32 epilogue (no cancellation in fp16)
// 16 warps = 4 per SM sub-partition, so each thread may use 128 registers (a 17th warp would cap it at 96).
constexpr int kGConsumerWarps = 15;
constexpr int kGConsumers = kGConsumerWarps * 32;     // 480
constexpr int kGThreads = kGConsumers + 32;           // + 1 producer warp = 512
constexpr int kGChunk = kGConsumers * 16;             // 7680 B: one 16-byte vector per consumer thread
constexpr int kGChunkElems = kGChunk / 2;             // 3840 bf16
constexpr int kGRing = 27;                            // 207 KB staging ring
constexpr int kGBarConsumers = 1;
constexpr int kRegChunks = 20;  // 20 x 3840 bf16 per CTA: V <= 153600 (Qwen: 151936 / 152064)

struct __align__(128) ClusterRegSmem {
  uint8_t ring[kGRing][kGChunk];
  uint64_t full[kGRing];
  uint64_t empty[kGRing];
  uint64_t xbar[2];
  uint4 xbuf[2];
  float red_m[kGConsumerWarps];
  float red_s[kGConsumerWarps];
  float za;
  float coef;
  float lse;
  float da;  // gradient at the action column, c (1 - p_a)
};

template <bool kStoreExp>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGThreads, 1)
    policy_loss_cluster_reg_kernel(const LossParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ClusterRegSmem& sm = *reinterpret_cast<ClusterRegSmem*>(smem_raw);
  const uint32_t rank = cluster_ctarank();
  const uint32_t cid = cluster_id_x(), ncl = nclusters_x();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int32_t V = p.V;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;
  const int32_t c0 = rank ? min(h, V) : 0;
  const int32_t c1 = rank ? V : min(h, V);
  const int32_t c1r = (c1 + 7) & ~7;
  const uint32_t slice_bytes = (uint32_t)(c1r - c0) * 2u;
  const int nchunks = (int)((slice_bytes + kGChunk - 1) / kGChunk);

  if (tid == 0) {
    for (int i = 0; i < kGRing; ++i) {
      mbar_init(smem_u32(&sm.full[i]), 1);
      mbar_init(smem_u32(&sm.empty[i]), kGConsumerWarps);
    }
    mbar_init(smem_u32(&sm.xbar[0]), 1);
    mbar_init(smem_u32(&sm.xbar[1]), 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();

  if (warp == kGConsumerWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t q = 0;
      for (int64_t row = cid; row < p.n_rows; row += ncl) {
        const uint8_t* src = p.logits + row * p.ld_bytes + (int64_t)c0 * 2;
        for (int c = 0; c < nchunks; ++c, ++q) {
          const uint32_t slot = q % kGRing, round = q / kGRing;
          mbar_wait(smem_u32(&sm.empty[slot]), (round & 1) ^ 1);
          const uint32_t nb = min((uint32_t)kGChunk, slice_bytes - (uint32_t)c * kGChunk);
          mbar_arrive_expect_tx(smem_u32(&sm.full[slot]), nb);
          bulk_g2s(smem_u32(&sm.ring[slot][0]), src + (int64_t)c * kGChunk, nb, smem_u32(&sm.full[slot]), pol);
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
    const int32_t col_t = c0 + tid * 8;  // this thread's first column; chunk c adds c * kGChunkElems
    // vectors this thread owns that lie inside the loaded bytes (all chunks but possibly the last)
    const int nvalid = nchunks - ((uint32_t)(nchunks - 1) * kGChunk + (uint32_t)tid * 16u >= slice_bytes ? 1 : 0);
    // the one vector straddling c1 when V % 8 != 0 (rank 1 only): chunk index, or -1
    const int tail_c = (c1 & 7) && ((c1 & ~7) - col_t) % kGChunkElems == 0 && (c1 & ~7) >= col_t
                           ? ((c1 & ~7) - col_t) / kGChunkElems : -1;
    const uint64_t l2e2 = f2(kLog2e, kLog2e);
    uint8_t* const logits = p.logits;
    uint32_t q = 0, it = 0;
    for (int64_t row = cid; row < p.n_rows; row += ncl, ++it) {
      const int32_t a = p.tok_action[row];
      RowMeta meta{0.f, 0.f, 0.f};
      if (tid == 0) meta = load_meta(p, row);

      // ---- pass 1a: ring -> registers; the slot is released at once (the producer refills it)
      uint4 v[kRegChunks];
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        v[c] = make_uint4(kBf16NegInf2, kBf16NegInf2, kBf16NegInf2, kBf16NegInf2);
        if (c < nchunks) {
          const uint32_t slot = q % kGRing, round = q / kGRing;
          ++q;
          mbar_wait(smem_u32(&sm.full[slot]), round & 1);
          const uint4 w = lds_v4(smem_u32(&sm.ring[slot][tid * 16]));
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&sm.empty[slot]));
          if (c < nvalid) v[c] = w;
        }
      }
      if (tail_c >= 0) {  // mask the columns >= V of the straddling vector (rare: V % 8 != 0)
        const int nkeep = c1 & 7;
#pragma unroll
        for (int c = 0; c < kRegChunks; ++c)
          if (c == tail_c) {
            uint32_t* w = &v[c].x;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e >= nkeep) w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0x0000FFFFu) | 0xFF800000u)
                                                  : ((w[e >> 1] & 0xFFFF0000u) | 0x0000FF80u);
          }
      }
      // running max over the thread's values (packed bf16 max is exact)
      uint32_t mx2 = kBf16NegInf2;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) mx2 = bmax2(mx2, bmax2(bmax2(v[c].x, v[c].y), bmax2(v[c].z, v[c].w)));
      const float mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u));
      // the action logit, from the owning thread's registers
      if (a >= col_t && a < c1 && ((a - col_t) % kGChunkElems) < 8) {
        const int ca = (a - col_t) / kGChunkElems, ea = (a - col_t) % kGChunkElems;
        uint32_t word = 0;
#pragma unroll
        for (int c = 0; c < kRegChunks; ++c)
          if (c == ca) word = (ea >> 1) == 0 ? v[c].x : (ea >> 1) == 1 ? v[c].y : (ea >> 1) == 2 ? v[c].z : v[c].w;
        sm.za = (ea & 1) ? __uint_as_float(word & 0xFFFF0000u) : __uint_as_float(word << 16);
      }

      // ---- pass 1b: e = 2^((z - m_t) log2e), s_t = sum e (two fp32 lanes); kStoreExp: v[c] <- e as fp16
      const float mb = (mx == -INFINITY) ? 0.0f : mx * kLog2e;
      const uint64_t nmb2 = f2(-mb, -mb);
      uint64_t s2 = f2(0.0f, 0.0f);
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        if (c < nchunks) {
          uint32_t* w = &v[c].x;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float e0, e1;
            f2split(fma2(bf2_to_f2(w[k]), l2e2, nmb2), e0, e1);
            e0 = ex2(e0);
            e1 = ex2(e1);
            s2 = add2(s2, f2(e0, e1));
            if (kStoreExp) w[k] = pack_f16x2(e0, e1);
          }
        }
      }
      float slo, shi;
      f2split(s2, slo, shi);
      MaxSum acc = warp_maxsum(MaxSum{mx, slo + shi});
      if (lane == 0) {
        sm.red_m[warp] = acc.m;
        sm.red_s[warp] = acc.s;
      }
      named_bar_sync(kGBarConsumers, kGConsumers);

      // ---- CTA-pair merge through DSMEM + the scalar epilogue (thread 0 of each CTA)
      if (tid == 0) {
        MaxSum mine{sm.red_m[0], sm.red_s[0]};
        for (int w = 1; w < kGConsumerWarps; ++w) mine = maxsum_merge(mine, MaxSum{sm.red_m[w], sm.red_s[w]});
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
        const float pa = ex2(fmaf(za, kLog2e, -lse * kLog2e));
        sm.coef = r.coef;
        sm.lse = lse;
        sm.da = fmaf(-r.coef, pa, r.coef);
      }
      named_bar_sync(kGBarConsumers, kGConsumers);
      const float coef = sm.coef, lse = sm.lse;

      // ---- pass 2: gradient from registers, 16-byte stores in place
      //   kStoreExp:  d = e * k_t,  k_t = -c 2^((m_t - lse) log2e)      (one FMUL2 per two logits)
      //   otherwise:  d = -c 2^((z - lse) log2e)                          (recomputed from the logits)
      const uint64_t k2 = kStoreExp ? f2(mx == -INFINITY ? 0.0f : -coef * ex2((mx - lse) * kLog2e),
                                         mx == -INFINITY ? 0.0f : -coef * ex2((mx - lse) * kLog2e))
                                    : f2(-coef, -coef);
      const uint64_t nlse2 = f2(-lse * kLog2e, -lse * kLog2e);
      uint8_t* dst = logits + row * p.ld_bytes + (int64_t)col_t * 2;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        if (c < nchunks) {
          const uint32_t* w = &v[c].x;
          uint32_t o[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float d0, d1;
            if (kStoreExp) {
              f2split(mul2(f2(f16lo(w[k]), f16hi(w[k])), k2), d0, d1);
            } else {
              float t0, t1;
              f2split(fma2(bf2_to_f2(w[k]), l2e2, nlse2), t0, t1);
              f2split(mul2(f2(ex2(t0), ex2(t1)), k2), d0, d1);
            }
            o[k] = pack_bf16x2(d0, d1);
          }
          if (c < nvalid && c != tail_c)
            stg_v4_hint(dst + (int64_t)c * kGChunk, make_uint4(o[0], o[1], o[2], o[3]), st_pol);
          if (c == tail_c) {  // straddling vector: only the columns < V
            __nv_bfloat16* dd = reinterpret_cast<__nv_bfloat16*>(dst + (int64_t)c * kGChunk);
            for (int e = 0; e < (c1 & 7); ++e)
              dd[e] = __ushort_as_bfloat16((unsigned short)((e & 1) ? (o[e >> 1] >> 16) : (o[e >> 1] & 0xFFFFu)));
          }
        }
      }
      // the action column: c (1 - p_a) from the fp32 epilogue (overwrites the value just stored above;
      // same thread, same address => program order)
      if (a >= col_t && a < c1 && ((a - col_t) % kGChunkElems) < 8)
        reinterpret_cast<__nv_bfloat16*>(logits + row * p.ld_bytes)[a] = __float2bfloat16_rn(sm.da);
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

bool cluster_reg_supports(int32_t dtype, int32_t V) {
  if (dtype != ECHO_BF16) return false;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;
  const int64_t bytes = (int64_t)h * 2;
  return V >= 2 * 8 && (bytes + kGChunk - 1) / kGChunk <= kRegChunks;
}

// How many 2-CTA clusters of `fn` can be resident at once (GPC shapes may strand SMs).  The persistent grid
// is sized to exactly that, so the static row striding never leaves a cluster for a second wave.
static int max_active_clusters(const void* fn, int threads, size_t smem, int fallback) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * 4096);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
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

template <bool kStoreExp>
static cudaError_t launch_cluster_reg(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  const size_t smem = sizeof(ClusterRegSmem);
  const void* fn = (const void*)policy_loss_cluster_reg_kernel<kStoreExp>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t clusters = max_active_clusters(fn, kGThreads, smem, num_sms / 2);
  if (clusters > p.n_rows) clusters = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)(clusters * 2), 2, kGThreads, (int32_t)smem};
    return cudaSuccess;
  }
  policy_loss_cluster_reg_kernel<kStoreExp><<<(unsigned)(clusters * 2), kGThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_policy_loss(const LossParams& p, int32_t dtype, int algo, cudaStream_t stream, int num_sms,
                               LaunchShape* shape) {
  if (algo == ECHO_ALGO_CLUSTER_REG) return launch_cluster_reg<true>(p, stream, num_sms, shape);
  if (algo == ECHO_ALGO_CLUSTER_REG_EXACT) return launch_cluster_reg<false>(p, stream, num_sms, shape);
  if (algo == ECHO_ALGO_CLUSTER_SMEM) {
    const size_t smem = sizeof(ClusterSmem);
    const void* fn = (const void*)policy_loss_cluster_kernel;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t clusters = max_active_clusters(fn, kCThreads, smem, num_sms / 2);
    if (clusters > p.n_rows) clusters = p.n_rows;
    if (shape) {
      *shape = LaunchShape{(int32_t)(clusters * 2), 2, kCThreads, (int32_t)smem};
      return cudaSuccess;
    }
    policy_loss_cluster_kernel<<<(unsigned)(clusters * 2), kCThreads, smem, stream>>>(p);
    return cudaGetLastError();
  }
  int64_t grid = num_sms;
  if (grid > p.n_rows) grid = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)grid, 1, kRThreads, 0};
    return cudaSuccess;
  }
  if (dtype == ECHO_BF16)
    policy_loss_row_kernel<1><<<(unsigned)grid, kRThreads, 0, stream>>>(p);
  else
    policy_loss_row_kernel<0><<<(unsigned)grid, kRThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace echo
