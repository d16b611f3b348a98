// lmhead.cu -- f2: the LM head fused with the log-softmax-and-gather of (3), and the two epilogues of
// the training step through the LM head (lmhead_bwd.cu, abi.cu): D = dL/dz recomputed from h and W (kMode 2,
// echo_lmhead_dlogits) and the logits themselves stored as bf16 (kMode 3, echo_lmhead_logits).  The store modes
// write through a per-warp 32 x 64 shared-memory box and a TMA store when V % 8 == 0 (sustained at the power cap,
// 8192 x 151936 x 5120 logits: 9.81 instead of 9.95 ms with per-thread 16-byte stores, profiles/r3y_lmtma.jsonl).
//
// logp_t = z[t, a_t] - logsumexp_v z[t, v],  z = h W^T  (h: [N x d] bf16 hidden states, W: [V x d] bf16 LM-head
// weight).  The [N x V] logits are never written to HBM: the GEMM runs on the 5th-generation tensor cores with
// the accumulator tile in TMEM, and its epilogue reduces every 128 x 256 logits tile to per-row partials
// (max, sum of exp) and picks out z[t, a_t]; a small finalize kernel merges the partials of a row in vocab-tile
// order (deterministic).  Traffic per token: 8 B x V/256 of partials instead of 2 x 2V B of logits.
//
// lmhead_tile_kernel: persistent, one CTA per SM, 6 warps, warp-specialised:
//   warp 0 (one lane)  TMA producer: 2-D tensor-map tile loads (SWIZZLE_128B) of A = h[128 rows x 64 k] (16 KB)
//                      and B = W[256 rows x 64 k] (32 KB) into a 4-stage shared-memory ring (full/empty mbarriers)
//   warp 1             allocates 512 TMEM columns (two 128 x 256 fp32 accumulators); one lane issues
//                      tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16, bf16 -> fp32) four per stage and
//                      tcgen05.commit's the stage back to the producer and the finished accumulator to the epilogue
//   warps 2-5          epilogue: tcgen05.ld 32 columns at a time (thread = row = TMEM lane), online max / sum of
//                      exp2 over the tile's valid columns, z[t, a_t] when the action falls in the tile; partials
//                      to the workspace; the accumulator is released as soon as it has been read, so the MMA of
//                      the next tile overlaps this epilogue
// Tiles are rasterised in groups of G token tiles x all vocab tiles (column-major inside a group), so the CTAs in
// flight share a few vocab tiles of B and the group's A rows; G is sized so that the group's A rows take ~42 MB of L2
// (G = 32 pair tiles x 256 x 2560 bf16 at d = 2560, 16 at d = 5120; the env var ECHO_LM_GROUP overrides it for A/B).
//
// kPair (ECHO_LMHEAD_PAIR, the default): a 2-CTA cluster shares one 256 x 256 tile with tcgen05.mma.cta_group::2
// (M = 256): each CTA stages its own 128 token rows of A and HALF of the 256 vocab rows of B, the leader CTA's one
// thread issues the MMA over both CTAs' shared memory, and each CTA's TMEM receives its 128 rows.  B traffic from
// L2 per token halves.  The TMA loads of both CTAs complete on the leader's full barrier (.cta_group::2), the
// commits multicast to both CTAs' empty / accumulator-full barriers, and both epilogues release the accumulator
// on the leader's barrier.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "umma.cuh"

namespace echo {

namespace lm {
constexpr int kBM = 128, kBN = 256, kBK = 64, kUmmaK = 16;  // per-CTA token rows, tile vocab columns, K step
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

template <bool kPair>
struct Cfg {
  static constexpr int kCtas = kPair ? 2 : 1;
  static constexpr int kBRows = kBN / kCtas;             // vocab rows of B staged by each CTA
  static constexpr int kABytes = kBM * kBK * 2, kBBytes = kBRows * kBK * 2, kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = kPair ? 6 : 4;
  static constexpr int kTileRows = kBM * kCtas;          // token rows of a (pair) tile
};
constexpr int kTidRing = 4;  // tile ids in flight between the scheduler (leader producer) and the other roles
template <bool kPair>
struct Smem {
  using C = Cfg<kPair>;
  uint8_t a[C::kStages][C::kABytes];
  uint8_t b[C::kStages][C::kBBytes];
  uint64_t full[C::kStages], empty[C::kStages], tfull[2], tempty[2];
  uint64_t tid_full[kTidRing], tid_empty[kTidRing];
  uint32_t tile_id[kTidRing];
  uint32_t tmem_base;
  alignas(1024) uint8_t zstage[4][32 * 128];  // store modes: per-warp staging box, 32 rows x 64 bf16 (SWIZZLE_128B)
};
// consumers of a tile id: the leader's MMA thread, 4 epilogue warps per CTA, the peer's producer thread
template <bool kPair>
constexpr uint32_t tid_consumers() { return kPair ? 10u : 5u; }
template <bool kPair>
constexpr size_t smem_bytes() { return sizeof(Smem<kPair>) + 1024; }  // + SWIZZLE_128B 1024-B alignment slack

// Instruction descriptor, kind::f16: fp32 accumulate (bits 4-5 = 1), A and B bf16 (bits 7-9, 10-12 = 1), both
// K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28 (M = 128 per CTA, 256 for the pair).
template <bool kPair>
constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) | ((uint32_t)((kBM * (kPair ? 2 : 1)) >> 4) << 24);
}

template <bool kPair>
ECHO_DEVINL void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  umma_f16<kPair>(tmem_d, adesc, bdesc, idesc<kPair>(), accumulate);
}
// tile u -> (token tile, vocab tile): groups of group_m token tiles, vocab-major inside a group
ECHO_DEVINL void tile_coords(int64_t u, int32_t n_tt, int32_t n_vt, int32_t group_m, int32_t& tt, int32_t& vt) {
  const int64_t per_group = (int64_t)group_m * n_vt;
  const int32_t g = (int32_t)(u / per_group);
  const int32_t rows_in_g = min(group_m, n_tt - g * group_m);
  const int64_t r = u - (int64_t)g * per_group;
  vt = (int32_t)(r / rows_in_g);
  tt = g * group_m + (int32_t)(r % rows_in_g);
}
}  // namespace lm

struct LmParams {
  int64_t n_rows;
  int32_t d, V, n_tt, n_vt, n_kb;
  int32_t group_m;  // token tiles per rasterisation group (launch_tile)
  int32_t pol;      // L2 hints on the operand loads (pair tile): 0 none, 1 h evict_last, 2 W evict_last (ECHO_LM_POL)
  int32_t tma_z;    // store modes: the bf16 output goes through map_z (TMA stores of 32 x 64 boxes)
  unsigned int* sched;  // this launch's {tile counter, finished CTAs} (in-order dynamic scheduler; reset by the last CTA)
  const int32_t* __restrict__ tok_action;
  float* __restrict__ part_m;  // [n_vt][n_rows]
  float* __restrict__ part_s;  // [n_vt][n_rows]
  float* __restrict__ part_t;  // [n_vt][n_rows]: sum z e^{z - m} (entropy output only)
  float* __restrict__ za;      // [n_rows]
  // dlogits mode (echo_lmhead_dlogits): per-row inputs and the bf16 output D [n_rows x ld]
  const float* __restrict__ g_lse;
  const float* __restrict__ g_coef;
  const float* __restrict__ g_ecoef;    // nullable: no entropy term
  const float* __restrict__ g_entropy;  // read iff g_ecoef
  uint16_t* __restrict__ dz;
  int64_t ld;
};

// kMode: 0 = logp partials, 1 = logp + entropy partials, 2 = dlogits (D written to p.dz), 3 = logits (z to p.dz)
// Tiles are handed out in order by a dynamic scheduler (as in gemm.cu): the leader's producer thread takes the next
// tile from a per-launch counter and broadcasts it to its MMA / epilogue warps and to the peer CTA through a 4-deep
// ring, so all clusters work inside one compact window of tiles.  (A static stride lets clusters drift apart over the
// ~1000 waves of a 32768-row launch, and the raster group's operands stop being shared in L2.)
template <bool kPair, int kMode>
__global__ void __launch_bounds__(lm::kThreads, 1)
    lmhead_tile_kernel(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_w,
                       const __grid_constant__ CUtensorMap map_z, const LmParams p) {
  using namespace lm;
  constexpr bool kEnt = kMode == 1, kStore = kMode >= 2;  // 2: D, 3: the logits z themselves (bf16)
  using C = Cfg<kPair>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  Smem<kPair>& sm = *reinterpret_cast<Smem<kPair>*>(smem_raw + (((raw + 1023u) & ~1023u) - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (int64_t)p.n_tt * p.n_vt;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  // tile id of the `use`-th tile of this cluster (every role walks the same sequence); n_tiles marks the end
  auto next_tile = [&](uint32_t use) -> int64_t {
    const uint32_t r = use % kTidRing, ph = (use / kTidRing) & 1u;
    mbar_wait_cluster(smem_u32(&sm.tid_full[r]), ph);
    return (int64_t)sm.tile_id[r];
  };
  auto next_tile_warp = [&](uint32_t use) -> int64_t {  // a whole warp: lane 0 polls, every lane then acquires
    const uint32_t r = use % kTidRing, ph = (use / kTidRing) & 1u;
    mbar_wait_cluster_warp(smem_u32(&sm.tid_full[r]), ph, lane);
    return (int64_t)sm.tile_id[r];
  };
  auto release_tile = [&](uint32_t use) {  // one arrival per consumer (thread or warp lane 0) on the leader
    const uint32_t r = use % kTidRing;
    if (leader) mbar_arrive(smem_u32(&sm.tid_empty[r]));
    else mbar_arrive_cluster(mapa(smem_u32(&sm.tid_empty[r]), 0));
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&sm.full[s]), 1);
      mbar_init(smem_u32(&sm.empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.tfull[b]), 1);
      mbar_init(smem_u32(&sm.tempty[b]), 4 * C::kCtas);  // one arrival per epilogue warp (of both CTAs)
    }
    for (int r = 0; r < kTidRing; ++r) {
      mbar_init(smem_u32(&sm.tid_full[r]), 1);
      mbar_init(smem_u32(&sm.tid_empty[r]), tid_consumers<kPair>());  // used on the leader only
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_h)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // barrier inits and TMEM allocation visible to the peer
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (the leader's is the scheduler)
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      const uint64_t pol_h = p.pol == 1 ? policy_evict_last() : policy_evict_normal();
      const uint64_t pol_w = p.pol == 2 ? policy_evict_last() : policy_evict_normal();
      for (uint32_t use = 0;; ++use) {
        int64_t u;
        if (leader) {
          const uint32_t r = use % kTidRing, ph = (use / kTidRing) & 1u;
          mbar_wait(smem_u32(&sm.tid_empty[r]), ph ^ 1u);
          u = (int64_t)atomicAdd(&p.sched[0], 1u);
          if (u > n_tiles) u = n_tiles;
          sm.tile_id[r] = (uint32_t)u;
          mbar_arrive(smem_u32(&sm.tid_full[r]));
          if constexpr (kPair) {
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa(smem_u32(&sm.tile_id[r]), 1)), "r"((uint32_t)u)
                         : "memory");
            mbar_arrive_cluster(mapa(smem_u32(&sm.tid_full[r]), 1));
          }
        } else {
          u = next_tile(use);
          release_tile(use);
        }
        if (u >= n_tiles) break;
        int32_t tt, vt;
        tile_coords(u, p.n_tt, p.n_vt, p.group_m, tt, vt);
        for (int32_t kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait(smem_u32(&sm.empty[stage]), phase ^ 1u);
          // both CTAs' bytes complete on the leader's full barrier; only the leader arms it (with both halves)
          const uint32_t bar = kPair ? mapa(smem_u32(&sm.full[stage]), 0) : smem_u32(&sm.full[stage]);
          if (leader) mbar_arrive_expect_tx(smem_u32(&sm.full[stage]), C::kStageBytes * C::kCtas);
          if (kPair && p.pol) {
            tma_load_2d_pair_hint(smem_u32(sm.a[stage]), &map_h, kb * kBK, tt * C::kTileRows + (int32_t)rank * kBM, bar,
                                  pol_h);
            tma_load_2d_pair_hint(smem_u32(sm.b[stage]), &map_w, kb * kBK, vt * kBN + (int32_t)rank * C::kBRows, bar,
                                  pol_w);
          } else {
            tma_load_2d<kPair>(smem_u32(sm.a[stage]), &map_h, kb * kBK, tt * C::kTileRows + (int32_t)rank * kBM, bar);
            tma_load_2d<kPair>(smem_u32(sm.b[stage]), &map_w, kb * kBK, vt * kBN + (int32_t)rank * C::kBRows, bar);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && leader) {  // pair: the leader's thread issues for both CTAs
      uint32_t stage = 0, phase = 0;
      for (uint32_t tc = 0;; ++tc) {
        const int64_t u = next_tile(tc);
        release_tile(tc);
        if (u >= n_tiles) break;
        const uint32_t buf = tc & 1u, aph = (tc >> 1) & 1u;
        mbar_wait_cluster(smem_u32(&sm.tempty[buf]), aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + buf * kBN;
        for (int32_t kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait_cluster(smem_u32(&sm.full[stage]), phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sm.a[stage]), b0 = smem_u32(sm.b[stage]);
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k)
            umma_bf16<kPair>(d_tmem, sw128_desc(a0 + k * kUmmaK * 2), sw128_desc(b0 + k * kUmmaK * 2),
                             (kb > 0 || k > 0) ? 1u : 0u);
          umma_commit<kPair>(smem_u32(&sm.empty[stage]));  // the stage's smem is free once these MMAs have read it
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit<kPair>(smem_u32(&sm.tfull[buf]));  // accumulator complete
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5 = TMEM lane quadrants)
    const int quad = warp & 3;
    uint32_t tc = 0;
    const uint32_t tempty_leader = kPair ? mapa(smem_u32(&sm.tempty[0]), 0) : smem_u32(&sm.tempty[0]);
    for (;; ++tc) {
      const int64_t u = next_tile_warp(tc);
      __syncwarp();
      if (lane == 0) release_tile(tc);
      if (u >= n_tiles) break;
      int32_t tt, vt;
      tile_coords(u, p.n_tt, p.n_vt, p.group_m, tt, vt);
      const uint32_t buf = tc & 1u, aph = (tc >> 1) & 1u;
      const int64_t row = (int64_t)tt * C::kTileRows + (int64_t)rank * kBM + quad * 32 + lane;
      const bool row_ok = row < p.n_rows;
      const int32_t a = (row_ok && kMode != 3) ? p.tok_action[row] : -1;
      const int32_t col0 = vt * kBN;
      if constexpr (kStore) {
        // D[t, v] = c (delta_{v,a} - p) + e p (z - lse + H) = p (e z + k) + c delta_{v,a},  k = e (H - lse) - c
        const bool rd = row_ok && kMode == 2;
        const float lse = rd ? p.g_lse[row] : 0.0f, c = rd ? p.g_coef[row] : 0.0f;
        const float e = (rd && p.g_ecoef) ? p.g_ecoef[row] : 0.0f;
        const float H = (rd && p.g_ecoef) ? p.g_entropy[row] : 0.0f;
        const float k = fmaf(e, H - lse, -c);
        const uint64_t l2e2 = f2(kLog2e, kLog2e), nl2 = f2(-lse * kLog2e, -lse * kLog2e), e2 = f2(e, e), k2 = f2(k, k);
        uint16_t* drow = p.dz + (row_ok ? row : 0) * p.ld;
        // one 32-column TMEM chunk -> 16 packed bf16 pairs (the logits, or D)
        auto convert = [&](const uint32_t (&r)[32], uint32_t (&o)[16], int32_t cb) {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            if constexpr (kMode == 3) {
              o[i >> 1] = pack_bf16x2(__uint_as_float(r[i]), __uint_as_float(r[i + 1]));
              continue;
            }
            const uint64_t z2 = f2(__uint_as_float(r[i]), __uint_as_float(r[i + 1]));
            float t0, t1;
            f2split(fma2(z2, l2e2, nl2), t0, t1);
            float d0, d1;
            f2split(mul2(f2(ex2(t0), ex2(t1)), fma2(z2, e2, k2)), d0, d1);
            if (cb + i == a) d0 += c;
            if (cb + i + 1 == a) d1 += c;
            o[i >> 1] = pack_bf16x2(d0, d1);
          }
        };
        mbar_wait_cluster_warp(smem_u32(&sm.tfull[buf]), aph, lane);
        tc_fence_after();
        if (p.tma_z) {
          // two chunks per 32 x 64 box in the warp's staging buffer (16-byte granule j of row r at j ^ (r & 7):
          // SWIZZLE_128B), written by one TMA store; the tensor map clips rows >= n_rows and columns >= V
          const int64_t row0 = row - lane;
          const uint32_t zst = smem_u32(sm.zstage[quad]);
#pragma unroll 1
          for (int c2 = 0; c2 < kBN / 64; ++c2) {
            const int32_t cbb = col0 + c2 * 64;
            if (cbb >= p.V || row0 >= p.n_rows) break;  // warp-uniform
            if (lane == 0) bulk_wait_read0();              // the box's previous contents have been read by the TMA
            __syncwarp();
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t r[32], o[16];
              tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + buf * kBN + c2 * 64 + hf * 32, r);
              convert(r, o, cbb + hf * 32);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                sts_v4(zst + (uint32_t)lane * 128u + ((uint32_t)((hf * 4 + j) ^ (lane & 7)) << 4),
                       make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]));
            }
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&map_z, zst, cbb, (int32_t)row0);
              bulk_commit();
            }
          }
        }
#pragma unroll 1
        for (int ch = 0; ch < (p.tma_z ? 0 : kBN / 32); ++ch) {
          const int32_t cb = col0 + ch * 32;
          if (cb >= p.V) break;  // warp-uniform: nothing left of the vocabulary in this tile
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + buf * kBN + ch * 32, r);
          uint32_t o[16];
          convert(r, o, cb);
          if (row_ok) {
            if (cb + 32 <= p.V) {
              uint4* dst = reinterpret_cast<uint4*>(drow + cb);
#pragma unroll
              for (int j = 0; j < 4; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (cb + i < p.V) drow[cb + i] = (uint16_t)((i & 1) ? (o[i >> 1] >> 16) : (o[i >> 1] & 0xFFFFu));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair) mbar_arrive_cluster(tempty_leader + buf * 8u);
          else mbar_arrive(smem_u32(&sm.tempty[buf]));
        }
        continue;
      }
      mbar_wait_cluster_warp(smem_u32(&sm.tfull[buf]), aph, lane);
      tc_fence_after();
      float m = -INFINITY, s = 0.0f, t = 0.0f, za = 0.0f;
      bool found = false;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + buf * kBN + c * 32, r);
        const int32_t cb = col0 + c * 32;
        if (cb + 32 > p.V) {  // the vocabulary's last, partial chunk: columns >= V do not exist
#pragma unroll
          for (int i = 0; i < 32; ++i)  // -inf (-1e30 with the entropy sum, so that e z is 0, not NaN)
            if (cb + i >= p.V) r[i] = kEnt ? 0xF149F2CAu : 0xFF800000u;
        }
        if ((uint32_t)(a - cb) < 32u) {  // the action's column is in this chunk (one chunk in ~4700)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cb + i == a) za = __uint_as_float(r[i]);
          found = true;
        }
        float cm = __uint_as_float(r[0]);
#pragma unroll
        for (int i = 1; i < 32; ++i) cm = fmaxf(cm, __uint_as_float(r[i]));
        if (cm > m) {
          const float f = (m == -INFINITY) ? 0.0f : ex2((m - cm) * kLog2e);
          s *= f;
          if (kEnt) t *= f;
          m = cm;
        }
        if (m != -INFINITY) {
          // 2^(z log2e - m log2e), packed fp32x2 FMA / add, one MUFU per logit
          const uint64_t nmb2 = f2(-m * kLog2e, -m * kLog2e), l2e2 = f2(kLog2e, kLog2e);
          uint64_t acc2 = f2(0.0f, 0.0f), acct = f2(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t z2 = f2(__uint_as_float(r[i]), __uint_as_float(r[i + 1]));
            float e0, e1;
            f2split(fma2(z2, l2e2, nmb2), e0, e1);
            const uint64_t e2 = f2(ex2(e0), ex2(e1));
            acc2 = add2(acc2, e2);
            if (kEnt) acct = fma2(e2, z2, acct);
          }
          float lo, hi;
          f2split(acc2, lo, hi);
          s += lo + hi;
          if (kEnt) {
            f2split(acct, lo, hi);
            t += lo + hi;
          }
        }
      }
      // accumulator read out: hand it back to the MMA warp before the global writes
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair) mbar_arrive_cluster(tempty_leader + buf * 8u);
        else mbar_arrive(smem_u32(&sm.tempty[buf]));
      }
      if (row_ok) {
        p.part_m[(int64_t)vt * p.n_rows + row] = m;
        p.part_s[(int64_t)vt * p.n_rows + row] = s;
        if (kEnt) p.part_t[(int64_t)vt * p.n_rows + row] = t;
        if (found) p.za[row] = za;
      }
    }
  }

  if constexpr (kStore) {
    if (warp >= 2 && p.tma_z && lane == 0) bulk_wait0();  // staging boxes read and stores done before the CTA retires
  }
  __syncwarp();
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
  if (threadIdx.x == 0) {  // every scheduler of this launch is done once all CTAs are here: reset the slot
    __threadfence();
    if (atomicAdd(&p.sched[1], 1u) == gridDim.x - 1) {
      p.sched[0] = 0u;
      p.sched[1] = 0u;
      __threadfence();
    }
  }
}

// One thread per row: merge the row's vocab-tile partials in tile order (deterministic), then logp = z_a - lse
// and, with tok_entropy, H = lse - (sum z e) / (sum e).
__global__ void __launch_bounds__(256) lmhead_finalize_kernel(int64_t n_rows, int32_t V, int32_t n_vt,
                                                              const int32_t* __restrict__ tok_action,
                                                              const float* __restrict__ part_m,
                                                              const float* __restrict__ part_s,
                                                              const float* __restrict__ part_t,
                                                              const float* __restrict__ za, float* __restrict__ tok_logp,
                                                              float* __restrict__ tok_lse,
                                                              float* __restrict__ tok_entropy) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= n_rows) return;
  float m = -INFINITY, s = 0.0f, t = 0.0f;
  for (int32_t vt = 0; vt < n_vt; ++vt) {
    const float mi = part_m[(int64_t)vt * n_rows + row], si = part_s[(int64_t)vt * n_rows + row];
    const float mm = fmaxf(m, mi);
    if (mm == -INFINITY) continue;
    const float fa = m == -INFINITY ? 0.0f : ex2((m - mm) * kLog2e);
    const float fb = mi == -INFINITY ? 0.0f : ex2((mi - mm) * kLog2e);
    s = s * fa + si * fb;
    if (tok_entropy) t = t * fa + part_t[(int64_t)vt * n_rows + row] * fb;
    m = mm;
  }
  const float lse = m + logf(s);
  const int32_t a = tok_action[row];
  tok_logp[row] = (a >= 0 && a < V) ? za[row] - lse : NAN;
  if (tok_lse) tok_lse[row] = lse;
  if (tok_entropy) tok_entropy[row] = lse - t / s;
}

// ------------------------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 2-D bf16 tensor map: `outer` rows of `inner` contiguous elements, row stride in bytes, SWIZZLE_128B boxes of
// box_inner (64: 128 B) x box_outer; out-of-bounds elements are zero-filled.
bool make_tensor_map_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                          uint32_t box_inner, uint32_t box_outer) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  // L2 sector promotion of the tensor-map loads: 256 B by default; ECHO_TMA_PROMO=0/1/2 (none / 64 B / 128 B) for A/B
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (const char* env = getenv("ECHO_TMA_PROMO")) {
    const int v = atoi(env);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
          : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tensor_map_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                         uint32_t box_inner, uint32_t box_outer) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map(CUtensorMap* map, const void* base, int64_t rows, int32_t d, uint32_t box_rows) {
  return make_tensor_map_bf16(map, base, (uint64_t)d, (uint64_t)rows, (uint64_t)d * 2, (uint32_t)lm::kBK, box_rows);
}

size_t lmhead_workspace_bytes(int64_t n_rows, int32_t V) {
  const int64_t n_vt = (V + lm::kBN - 1) / lm::kBN;
  return (size_t)(3 * n_vt + 1) * (size_t)n_rows * sizeof(float);
}

#ifdef ECHO_LMHEAD_SINGLE
constexpr bool kLmPair = false;
#else
constexpr bool kLmPair = true;
#endif

// In-order dynamic tile scheduler slots (as in gemm.cu): one {counter, finished CTAs} pair per launch, reset by the
// launch's last CTA; graph-captured launches keep theirs (next_sched_slot).
constexpr int kLmSlots = 64;
__device__ unsigned int g_lm_sched[kLmSlots][2];
static std::atomic<uint32_t> g_lm_next_slot{0}, g_lm_next_slot_graph{0};

// Persistent launch of lmhead_tile_kernel<kLmPair, kMode>: one (pair) cluster per resident slot, capped at the tile
// count.  p's shape fields are filled in here.
template <int kMode>
static cudaError_t launch_tile(const void* hidden, const void* weight, LmParams& p, cudaStream_t stream, int num_sms) {
  using C = lm::Cfg<kLmPair>;
  CUtensorMap mh, mw;
  if (!make_map(&mh, hidden, p.n_rows, p.d, lm::kBM) || !make_map(&mw, weight, p.V, p.d, C::kBRows))
    return cudaErrorInvalidValue;
  p.n_tt = (int32_t)((p.n_rows + C::kTileRows - 1) / C::kTileRows);
  p.n_vt = (p.V + lm::kBN - 1) / lm::kBN;
  p.n_kb = (p.d + lm::kBK - 1) / lm::kBK;
  // group A rows ~42 MB: 16 / 32 / 64 / 128 pair tiles A/B'd at d = 2560 on the 32768-row logp launch, 32 fastest;
  // 4 / 8 / 16 / 32 at d = 5120: 16 fastest (profiles/r2i_ab_knobs.jsonl)
  p.group_m = (int32_t)((42ll << 20) / ((int64_t)C::kTileRows * p.d * 2));
  if (const char* env = getenv("ECHO_LM_GROUP")) p.group_m = atoi(env);
  p.group_m = p.group_m < 2 ? 2 : p.group_m > 128 ? 128 : p.group_m;
  p.pol = 0;
  if (const char* env = getenv("ECHO_LM_POL")) p.pol = atoi(env);  // A/B knob: 1 h evict_last, 2 W evict_last
  const void* fn = (const void*)lmhead_tile_kernel<kLmPair, kMode>;
  const size_t smem = lm::smem_bytes<kLmPair>();
  // per device, once: the shared-memory opt-in and the resident-cluster count
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int64_t units = dev < 64 ? (int64_t)cached[dev].load(std::memory_order_relaxed) - 1 : -1;
  if (units < 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    units = kLmPair ? max_active_clusters(fn, lm::kThreads, smem, C::kCtas, num_sms / C::kCtas) : num_sms;
    if (dev < 64) cached[dev].store((int)units + 1, std::memory_order_relaxed);
  }
  const int64_t n_tiles = (int64_t)p.n_tt * p.n_vt;
  if (units > n_tiles) units = n_tiles;
  unsigned int* slots = nullptr;
  e = cudaGetSymbolAddress((void**)&slots, g_lm_sched);
  if (e != cudaSuccess) return e;
  p.sched = slots + 2 * next_sched_slot(g_lm_next_slot, g_lm_next_slot_graph, stream, kLmSlots);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * C::kCtas));
  cfg.blockDim = dim3(lm::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C::kCtas;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  // store modes: the bf16 output [n_rows x V] (row stride ld) through a tensor map when its base is 16-B aligned and
  // V % 8 == 0 (a tensor-map store writes whole 16-byte granules: a ragged last one would spill into columns >= V)
  CUtensorMap mz;
  memset(&mz, 0, sizeof(mz));
  p.tma_z = 0;
  if (kMode >= 2 && (reinterpret_cast<uintptr_t>(p.dz) & 15) == 0 && p.ld % 8 == 0 && p.V % 8 == 0)
    p.tma_z = make_tensor_map_bf16(&mz, p.dz, (uint64_t)p.V, (uint64_t)p.n_rows, (uint64_t)p.ld * 2, 64, 32) ? 1 : 0;
  if (const char* env = getenv("ECHO_LM_TMA_OUT")) p.tma_z = p.tma_z && atoi(env) != 0;  // A/B knob
  return cudaLaunchKernelEx(&cfg, lmhead_tile_kernel<kLmPair, kMode>, mh, mw, mz, p);
}

cudaError_t launch_lmhead_logp(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                               const int32_t* tok_action, float* tok_logp, float* tok_lse, float* tok_entropy,
                               void* workspace, cudaStream_t stream, int num_sms) {
  if (n_rows == 0) return cudaSuccess;
  LmParams p{};
  p.n_rows = n_rows;
  p.d = d;
  p.V = V;
  p.tok_action = tok_action;
  const int32_t n_vt = (V + lm::kBN - 1) / lm::kBN;
  float* ws = static_cast<float*>(workspace);
  p.part_m = ws;
  p.part_s = ws + (size_t)n_vt * n_rows;
  p.part_t = ws + (size_t)2 * n_vt * n_rows;
  p.za = ws + (size_t)3 * n_vt * n_rows;
  const cudaError_t e = tok_entropy ? launch_tile<1>(hidden, weight, p, stream, num_sms)
                                    : launch_tile<0>(hidden, weight, p, stream, num_sms);
  if (e != cudaSuccess) return e;
  lmhead_finalize_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, stream>>>(n_rows, V, n_vt, tok_action, p.part_m,
                                                                              p.part_s, p.part_t, p.za, tok_logp, tok_lse,
                                                                              tok_entropy);
  return cudaGetLastError();
}

cudaError_t launch_lmhead_dlogits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                  const int32_t* tok_action, const float* tok_lse, const float* tok_coef,
                                  const float* tok_ecoef, const float* tok_entropy, void* dlogits, int64_t ld,
                                  cudaStream_t stream, int num_sms) {
  if (n_rows == 0) return cudaSuccess;
  LmParams p{};
  p.n_rows = n_rows;
  p.d = d;
  p.V = V;
  p.tok_action = tok_action;
  p.g_lse = tok_lse;
  p.g_coef = tok_coef;
  p.g_ecoef = tok_ecoef;
  p.g_entropy = tok_entropy;
  p.dz = static_cast<uint16_t*>(dlogits);
  p.ld = ld;
  return launch_tile<2>(hidden, weight, p, stream, num_sms);
}

cudaError_t launch_lmhead_logits(const void* hidden, const void* weight, int64_t n_rows, int32_t d, int32_t V,
                                 void* logits, int64_t ld, cudaStream_t stream, int num_sms) {
  if (n_rows == 0) return cudaSuccess;
  LmParams p{};
  p.n_rows = n_rows;
  p.d = d;
  p.V = V;
  p.dz = static_cast<uint16_t*>(logits);
  p.ld = ld;
  return launch_tile<3>(hidden, weight, p, stream, num_sms);
}

}  // namespace echo
