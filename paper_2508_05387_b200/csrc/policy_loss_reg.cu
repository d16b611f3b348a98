// policy_loss_reg.cu -- ECHO_ALGO_CLUSTER_REG / _EXACT, the flagship kernel (see policy_loss.cu).
#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

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
  const uint32_t full0 = smem_u32(&sm.full[0]), empty0 = smem_u32(&sm.empty[0]), ring0 = smem_u32(&sm.ring[0][0]);

  if (tid == 0) {
    for (int i = 0; i < kGRing; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, kGConsumerWarps);
    }
    mbar_init(smem_u32(&sm.xbar[0]), 1);
    mbar_init(smem_u32(&sm.xbar[1]), 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();

  if (warp == kGConsumerWarps) {
    // ------------------------------------------------------------ producer: TMA bulk loads into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t slot = 0, phase = 0;
      for (int64_t row = cid; row < p.n_rows; row += ncl) {
        const uint8_t* src = p.logits + row * p.ld_bytes + (int64_t)c0 * 2;
        for (int c = 0; c < nchunks; ++c) {
          mbar_wait(empty0 + 8 * slot, phase ^ 1);
          const uint32_t nb = min((uint32_t)kGChunk, slice_bytes - (uint32_t)c * kGChunk);
          mbar_arrive_expect_tx(full0 + 8 * slot, nb);
          bulk_g2s(ring0 + slot * kGChunk, src + (int64_t)c * kGChunk, nb, full0 + 8 * slot, pol);
          if (++slot == kGRing) {
            slot = 0;
            phase ^= 1;
          }
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
    const float gscale = (float)((double)p.grad_scale / *p.n_global);  // c_t = dl/dlogp * (s / N_global)
    const int32_t col_t = c0 + tid * 8;  // this thread's first column; chunk c adds c * kGChunkElems
    // does this thread's vector of the last chunk lie inside the loaded bytes?
    const bool last_valid = (uint32_t)(nchunks - 1) * kGChunk + (uint32_t)tid * 16u < slice_bytes;
    // vector straddling c1 (V % 8 != 0, rank 1): it is this thread's last loaded vector
    const bool has_tail = (c1 & 7) && (c1 & ~7) >= col_t && ((c1 & ~7) - col_t) % kGChunkElems == 0;
    // full vectors this thread stores in pass 2: chunks [0, nstore)
    const int nstore = nchunks - (last_valid ? 0 : 1) - (has_tail ? 1 : 0);
    const uint64_t l2e2 = f2(kLog2e, kLog2e);
    const uint32_t my_off = (uint32_t)tid * 16u;
    uint32_t slot = 0, phase = 0, it = 0;
    for (int64_t row = cid; row < p.n_rows; row += ncl, ++it) {
      const int32_t a = p.tok_action[row];
      RowMeta meta{0.f, 0.f, 0.f};
      if (tid == 0) meta = load_meta(p, row);

      ECHO_TRACE_MARK(p, it, 0);
      // ---- pass 1a: ring -> registers, then release the row's slots (the producer refills them)
      uint4 v[kRegChunks];
      uint32_t rel_slot = slot;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        if (c < nchunks) {
          mbar_wait(full0 + 8 * slot, phase);
          uint4 w = lds_v4(ring0 + slot * kGChunk + my_off);
          if (c == nchunks - 1) {  // last chunk: beyond the loaded bytes -> -inf; straddling vector -> mask
            if (!last_valid) w = make_uint4(kBf16NegInf2, kBf16NegInf2, kBf16NegInf2, kBf16NegInf2);
            if (has_tail) w = mask_tail(w, c1 & 7);
          }
          v[c] = w;
          if (++slot == kGRing) {
            slot = 0;
            phase ^= 1;
          }
        } else {
          v[c] = make_uint4(kBf16NegInf2, kBf16NegInf2, kBf16NegInf2, kBf16NegInf2);
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < nchunks; ++c) {
          mbar_arrive(empty0 + 8 * rel_slot);
          if (++rel_slot == kGRing) rel_slot = 0;
        }
      }
      // running max over the thread's values (packed bf16 max is exact)
      ECHO_TRACE_MARK(p, it, 1);
      uint32_t mx2 = kBf16NegInf2;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) mx2 = bmax2(mx2, bmax2(bmax2(v[c].x, v[c].y), bmax2(v[c].z, v[c].w)));
      const float mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u));
      // the action logit, from the owning thread's registers
      const bool own_a = a >= col_t && a < c1 && ((a - col_t) % kGChunkElems) < 8;
      if (own_a) {
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
      ECHO_TRACE_MARK(p, it, 2);
      named_bar_sync(kGBarConsumers, kGConsumers);
      ECHO_TRACE_MARK(p, it, 3);

      // ---- CTA merge (warp 0, shuffle tree), CTA-pair merge through DSMEM, scalar epilogue (lane 0)
      if (warp == 0) {
        MaxSum mine = lane < kGConsumerWarps ? MaxSum{sm.red_m[lane], sm.red_s[lane]} : MaxSum{-INFINITY, 0.0f};
        mine = warp_maxsum(mine);
        if (lane == 0) {
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
          const RowScalars r = row_epilogue_f(lse, za, meta.old, meta.ref, meta.adv, p.clip_low, p.clip_high,
                                              p.kl_coef, gscale);
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
      }
      named_bar_sync(kGBarConsumers, kGConsumers);
      ECHO_TRACE_MARK(p, it, 4);
      const float coef = sm.coef, lse = sm.lse;

      // ---- pass 2: gradient from registers, 16-byte stores in place
      //   kStoreExp:  d = e * k_t,  k_t = -c 2^((m_t - lse) log2e)      (one FMUL2 per two logits)
      //   otherwise:  d = -c 2^((z - lse) log2e)                          (recomputed from the logits)
      const float kt = mx == -INFINITY ? 0.0f : -coef * ex2((mx - lse) * kLog2e);
      const uint64_t k2 = kStoreExp ? f2(kt, kt) : f2(-coef, -coef);
      const uint64_t nlse2 = f2(-lse * kLog2e, -lse * kLog2e);
      uint8_t* const row_base = p.logits + row * p.ld_bytes;
      uint8_t* const dst = row_base + (int64_t)col_t * 2;
#pragma unroll
      for (int c = 0; c < kRegChunks; ++c) {
        if (c < nchunks) {
          uint32_t* w = &v[c].x;
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
            w[k] = pack_bf16x2(d0, d1);
          }
          if (c < nstore) {
            stg_v4_hint(dst + (int64_t)c * kGChunk, v[c], st_pol);
          } else if (has_tail && c == nchunks - 1) {  // straddling vector: only the columns < V
            __nv_bfloat16* dd = reinterpret_cast<__nv_bfloat16*>(dst + (int64_t)c * kGChunk);
            const uint32_t ow[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e < (c1 & 7))
                dd[e] = __ushort_as_bfloat16((unsigned short)((e & 1) ? (ow[e >> 1] >> 16) : (ow[e >> 1] & 0xFFFFu)));
          }
        }
      }
      // the action column: c (1 - p_a) from the fp32 epilogue (overwrites the value just stored above;
      // same thread, same address => program order)
      ECHO_TRACE_MARK(p, it, 5);
      if (own_a) reinterpret_cast<__nv_bfloat16*>(row_base)[a] = __float2bfloat16_rn(sm.da);
    }
  }
  cluster_sync_all();
}


bool cluster_reg_supports(int32_t dtype, int32_t V) {
  if (dtype != ECHO_BF16) return false;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;
  const int64_t bytes = (int64_t)h * 2;
  return V >= 2 * 8 && (bytes + kGChunk - 1) / kGChunk <= kRegChunks;
}

template <bool kStoreExp>
static cudaError_t launch_cluster_reg_t(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  const size_t smem = sizeof(ClusterRegSmem);
  const void* fn = (const void*)policy_loss_cluster_reg_kernel<kStoreExp>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t clusters = max_active_clusters(fn, kGThreads, smem, 2, num_sms / 2);
  if (clusters > p.n_rows) clusters = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)(clusters * 2), 2, kGThreads, (int32_t)smem};
    return cudaSuccess;
  }
  policy_loss_cluster_reg_kernel<kStoreExp><<<(unsigned)(clusters * 2), kGThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_cluster_reg(const LossParams& p, bool store_exp, cudaStream_t stream, int num_sms,
                               LaunchShape* shape) {
  return store_exp ? launch_cluster_reg_t<true>(p, stream, num_sms, shape)
                   : launch_cluster_reg_t<false>(p, stream, num_sms, shape);
}

}  // namespace echo
