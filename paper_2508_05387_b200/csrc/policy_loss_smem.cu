// policy_loss_smem.cu -- ECHO_ALGO_CLUSTER_SMEM (see policy_loss.cu for the overview).
#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

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

bool cluster_algo_supports(int32_t dtype, int32_t V) {
  if (dtype != ECHO_BF16) return false;
  const int32_t h = (((V + 1) >> 1) + 7) & ~7;
  const int64_t bytes = (int64_t)h * 2;
  return V >= 2 * 8 && (bytes + kCChunk - 1) / kCChunk <= kCMaxChunksPerRow;
}

cudaError_t launch_cluster_smem(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  const size_t smem = sizeof(ClusterSmem);
  const void* fn = (const void*)policy_loss_cluster_kernel;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t clusters = max_active_clusters(fn, kCThreads, smem, 2, num_sms / 2);
  if (clusters > p.n_rows) clusters = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)(clusters * 2), 2, kCThreads, (int32_t)smem};
    return cudaSuccess;
  }
  policy_loss_cluster_kernel<<<(unsigned)(clusters * 2), kCThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace echo
