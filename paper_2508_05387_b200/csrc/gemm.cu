// gemm.cu -- the two plain GEMMs of the f2 backward on the tcgen05 tensor cores:
//   dhidden = D W       C[t, j]  = sum_v D[t, v] W[v, j]     A = D  (K-major),  B = W (MN-major)
//   dweight (+)= D^T h  C[v, j] (+)= sum_t D[t, v] h[t, j]   A = D  (MN-major), B = h (MN-major)
// with D the bf16 [rows x ld] logits gradient of a chunk, W the bf16 [V x d] LM-head weight, h the bf16 [rows x d]
// hidden states, fp32 accumulation in TMEM and an fp32 output (overwritten or accumulated).
//
// gemm_tile_kernel<kAMN, kBMN>: C[m, n] = sum_k A(m, k) B(n, k), persistent 2-CTA clusters (cta_group::2), a pair
// tile of 256 (M, 128 per CTA) x 256 (N, 128 per CTA staged), K in steps of 64, 6-stage TMA ring, 2 TMEM accumulators
// (512 columns), warp-specialised like lmhead_tile_kernel (warp 0 TMA, warp 1 MMA, warps 2-5 epilogue).  Operands are
// K-major (global [M x K], K contiguous: one SWIZZLE_128B box of 64 K x 128 rows per stage) or MN-major (global
// [K x M], M contiguous: two boxes of 64 M x 64 K per stage; UMMA canonical MN-major SW128 layout with 1024-B atoms of
// 64 MN x 8 K, LBO = 8 KB between the two 64-wide MN atoms, SBO = 1 KB between 8-row K groups, +2 KB per K = 16
// step).  Epilogue: thread = output row (TMEM lane), 32 fp32 columns per tcgen05.ld, 16-byte stores (+ loads when
// accumulating).  Tiles are handed out in order by a dynamic scheduler (the leader's producer thread owns a per-launch
// counter and broadcasts tile ids to its MMA / epilogue warps and to the peer CTA through a 4-deep ring); a poorly
// filled last wave with a long K loop is avoided by a deterministic two-pass split-K (lower K halves first, the upper
// half's epilogue adds onto the lower half's stores after a per-tile counter says they are complete).
#include <cuda.h>
#include <cuda_bf16.h>

#include <atomic>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "umma.cuh"

namespace echo {

namespace gm {
constexpr int kBM = 128, kBN = 256, kBK = 64, kUmmaK = 16, kThreads = 192, kStages = 6;
constexpr int kOpBytes = 128 * kBK * 2;  // one operand's stage per CTA: 128 rows (M or N) x 64 K bf16 = 16 KB
constexpr uint32_t kTmemCols = 512;
constexpr int kTidRing = 4;  // tile ids in flight between the scheduler (leader producer) and the other roles
struct Smem {
  uint8_t a[kStages][kOpBytes];
  uint8_t b[kStages][kOpBytes];
  uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  uint64_t tid_full[kTidRing], tid_empty[kTidRing];
  uint32_t tile_id[kTidRing];
  uint32_t tmem_base;
};
// consumers of a tile id: the leader's MMA thread and 4 epilogue warps, the peer's producer thread and 4 epilogue warps
constexpr uint32_t kTidConsumers = 10;
constexpr size_t smem_bytes() { return sizeof(Smem) + 1024; }

// MN-major SWIZZLE_128B descriptor: start >> 4 | LBO 8192 B (>> 4) | SBO 1024 B (>> 4) | version 1 | layout 2
ECHO_DEVINL uint64_t sw128_mn_desc(uint32_t smem_addr) {
  return (uint64_t)((smem_addr & 0x3FFFFu) >> 4) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <bool kMN>
ECHO_DEVINL uint64_t op_desc(uint32_t base, int k) {  // descriptor of the k-th K = 16 slice of a stage
  return kMN ? sw128_mn_desc(base + k * (kUmmaK * 128)) : lm::sw128_desc(base + k * (kUmmaK * 2));
}
// kind::f16, fp32 accumulate, bf16 A / B, majors, N = 256, M = 256 (pair)
template <bool kAMN, bool kBMN>
constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)kAMN << 15) | ((uint32_t)kBMN << 16) |
         ((uint32_t)(kBN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
// stage one operand's 128 rows (M or N) x 64 K of this CTA
template <bool kMN>
ECHO_DEVINL void load_op(uint32_t dst, const CUtensorMap* map, int32_t row0, int32_t k0, uint32_t bar, uint64_t pol) {
  if constexpr (kMN) {  // global [K x rows]: two boxes {64 rows, 64 K}
    lm::tma_load_2d_pair_hint(dst, map, row0, k0, bar, pol);
    lm::tma_load_2d_pair_hint(dst + 8192, map, row0 + 64, k0, bar, pol);
  } else {              // global [rows x K]: one box {64 K, 128 rows}
    lm::tma_load_2d_pair_hint(dst, map, k0, row0, bar, pol);
  }
}
// tile u -> (M tile, N tile): groups of group_m M tiles x all N tiles, M-fastest inside a group.  The host sizes a
// group to about half a wave of clusters (group_m = clusters / (2 N tiles)), so the tiles in flight share their A rows
// and B columns k-block by k-block and each operand streams from DRAM about once per group.
ECHO_DEVINL void tile_coords(int64_t u, int32_t n_mt, int32_t n_nt, int32_t group_m, int32_t& mt, int32_t& nt) {
  const int64_t per_group = (int64_t)group_m * n_nt;
  const int32_t g = (int32_t)(u / per_group);
  const int32_t rows_in_g = min(group_m, n_mt - g * group_m);
  const int64_t r = u - (int64_t)g * per_group;
  nt = (int32_t)(r / rows_in_g);
  mt = g * group_m + (int32_t)(r % rows_in_g);
}
}  // namespace gm

// In-order dynamic tile scheduler: per-launch counter slots (round robin over kGemmSlots, each reset to zero by its
// launch's last CTA), so that clusters that start late or run slow take fewer tiles -- no wave-quantisation tail.
constexpr int kGemmSlots = 64;
__device__ unsigned int g_gemm_sched[kGemmSlots][2];
// split-K: per output tile, the number of epilogue warps (8) that have stored the lower K half (zeroed at teardown); the
// upper half of tile t has id n_out + t, so it is handed out after every lower half (in-order scheduler: no deadlock)
constexpr int kMaxSplitTiles = 4096;
__device__ unsigned int g_gemm_flags[kGemmSlots][kMaxSplitTiles];
static std::atomic<uint32_t> g_gemm_next_slot{0}, g_gemm_next_slot_graph{0};

struct GemmParams {
  int64_t M;
  int32_t N, K, n_mt, n_nt, n_kb, group_m;
  unsigned int* sched;  // this launch's {tile counter, finished CTAs} (reset by the last CTA)
  unsigned int* flags;  // split-K: this launch's per-output-tile counters
  int32_t split;        // 1 or 2: K halves per output tile (ids t, n_out + t: the second pass adds onto the first)
  int32_t pol_a, pol_b;  // L2 policy per operand: 2 = evict_last (small, re-read by every tile), 1 = evict_first
                         // (streamed past a kept operand), 0 = evict_normal
  float* __restrict__ out;
  int64_t ldo;
  int32_t accumulate;
};

template <bool kAMN, bool kBMN>
__global__ void __launch_bounds__(gm::kThreads, 1)
    gemm_tile_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const GemmParams p) {
  using namespace gm;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw + (((raw + 1023u) & ~1023u) - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_out = (int64_t)p.n_mt * p.n_nt, n_tiles = n_out * p.split;
  const int32_t kb_half = p.n_kb / 2;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // tile id of the `use`-th tile of this cluster (every role walks the same sequence); n_tiles marks the end
  auto next_tile = [&](uint32_t use) -> int64_t {
    const uint32_t r = use % kTidRing, ph = (use / kTidRing) & 1u;
    mbar_wait_cluster(smem_u32(&sm.tid_full[r]), ph);
    return (int64_t)sm.tile_id[r];
  };
  auto release_tile = [&](uint32_t use) {  // one arrival per consumer (thread or warp lane 0) on the leader
    const uint32_t r = use % kTidRing;
    if (leader) mbar_arrive(smem_u32(&sm.tid_empty[r]));
    else lm::mbar_arrive_cluster(mapa(smem_u32(&sm.tid_empty[r]), 0));
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&sm.full[s]), 1);
      mbar_init(smem_u32(&sm.empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&sm.tfull[b]), 1);
      mbar_init(smem_u32(&sm.tempty[b]), 8);  // one arrival per epilogue warp of both CTAs
    }
    for (int r = 0; r < kTidRing; ++r) {
      mbar_init(smem_u32(&sm.tid_full[r]), 1);
      mbar_init(smem_u32(&sm.tid_empty[r]), kTidConsumers);  // used on the leader only
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  lm::tc_fence_before();
  cluster_sync_all();
  lm::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      const uint64_t pol_a = p.pol_a == 2 ? policy_evict_last() : p.pol_a == 1 ? policy_evict_first()
                                                                                : policy_evict_normal();
      const uint64_t pol_b = p.pol_b == 2 ? policy_evict_last() : p.pol_b == 1 ? policy_evict_first()
                                                                                : policy_evict_normal();
      for (uint32_t use = 0;; ++use) {
        int64_t u;
        if (leader) {  // the scheduler: grab the next tile, publish it to this CTA and the peer
          const uint32_t r = use % kTidRing, ph = (use / kTidRing) & 1u;
          mbar_wait(smem_u32(&sm.tid_empty[r]), ph ^ 1u);
          u = (int64_t)atomicAdd(&p.sched[0], 1u);
          if (u > n_tiles) u = n_tiles;
          sm.tile_id[r] = (uint32_t)u;
          mbar_arrive(smem_u32(&sm.tid_full[r]));
          asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa(smem_u32(&sm.tile_id[r]), 1)), "r"((uint32_t)u)
                       : "memory");
          lm::mbar_arrive_cluster(mapa(smem_u32(&sm.tid_full[r]), 1));
        } else {
          u = next_tile(use);
          release_tile(use);
        }
        if (u >= n_tiles) break;
        int32_t mt, nt;
        const bool upper = u >= n_out;  // split-K: the second pass over the upper K half
        tile_coords(upper ? u - n_out : u, p.n_mt, p.n_nt, p.group_m, mt, nt);
        const int32_t m_row = mt * 256 + (int32_t)rank * kBM, n_row = nt * kBN + (int32_t)rank * 128;
        const int32_t kb0 = upper ? kb_half : 0;
        const int32_t kb1 = (p.split == 1 || upper) ? p.n_kb : kb_half;
        for (int32_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&sm.empty[stage]), phase ^ 1u);
          const uint32_t bar = mapa(smem_u32(&sm.full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(smem_u32(&sm.full[stage]), 4 * kOpBytes);
          load_op<kAMN>(smem_u32(sm.a[stage]), &map_a, m_row, kb * kBK, bar, pol_a);
          load_op<kBMN>(smem_u32(sm.b[stage]), &map_b, n_row, kb * kBK, bar, pol_b);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (the leader's lane 0)
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, tc = 0;
      for (;; ++tc) {
        const int64_t u = next_tile(tc);
        release_tile(tc);
        if (u >= n_tiles) break;
        const uint32_t buf = tc & 1u, aph = (tc >> 1) & 1u;
        mbar_wait_cluster(smem_u32(&sm.tempty[buf]), aph ^ 1u);
        lm::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * kBN;
        const bool upper = u >= n_out;
        const int32_t kb0 = upper ? kb_half : 0;
        const int32_t kb1 = (p.split == 1 || upper) ? p.n_kb : kb_half;
        for (int32_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait_cluster(smem_u32(&sm.full[stage]), phase);
          lm::tc_fence_after();
          const uint32_t a0 = smem_u32(sm.a[stage]), b0 = smem_u32(sm.b[stage]);
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k)
            lm::umma_f16<true>(d_tmem, op_desc<kAMN>(a0, k), op_desc<kBMN>(b0, k), idesc<kAMN, kBMN>(),
                               (kb > kb0 || k > 0) ? 1u : 0u);
          lm::umma_commit<true>(smem_u32(&sm.empty[stage]));
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        lm::umma_commit<true>(smem_u32(&sm.tfull[buf]));
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5 = TMEM lane quadrants)
    const int quad = warp & 3;
    uint32_t tc = 0;
    const uint32_t tempty_leader = mapa(smem_u32(&sm.tempty[0]), 0);
    const bool vec_ok = (p.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
    for (;; ++tc) {
      const int64_t u = next_tile(tc);
      __syncwarp();
      if (lane == 0) release_tile(tc);
      if (u >= n_tiles) break;
      int32_t mt, nt;
      const int64_t ot = u >= n_out ? u - n_out : u;  // output tile
      tile_coords(ot, p.n_mt, p.n_nt, p.group_m, mt, nt);
      const uint32_t buf = tc & 1u, aph = (tc >> 1) & 1u;
      const int64_t row = (int64_t)mt * 256 + (int64_t)rank * kBM + quad * 32 + lane;
      const bool row_ok = row < p.M;
      float* orow = p.out + (row_ok ? row : 0) * p.ldo;
      // split-K: the second half adds onto the first half's stores (fixed order: deterministic)
      const bool second = u >= n_out;
      const bool acc = p.accumulate || second;
      mbar_wait_cluster(smem_u32(&sm.tfull[buf]), aph);
      lm::tc_fence_after();
      if (second) {
        if (lane == 0) {
          uint32_t v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.flags + ot) : "memory");
          } while (v < 8u);
        }
        __syncwarp();
        __threadfence();
      }
#pragma unroll 1
      for (int ch = 0; ch < kBN / 32; ++ch) {
        const int32_t cb = nt * kBN + ch * 32;
        if (cb >= p.N) break;  // warp-uniform
        uint32_t r[32];
        lm::tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + buf * kBN + ch * 32, r);
        if (!row_ok) continue;
        if (vec_ok && cb + 32 <= p.N) {
          float4* dst = reinterpret_cast<float4*>(orow + cb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            if (acc) {
              const float4 o = __ldcg(dst + j);
              v.x += o.x;
              v.y += o.y;
              v.z += o.z;
              v.w += o.w;
            }
            dst[j] = v;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cb + i < p.N) orow[cb + i] = __uint_as_float(r[i]) + (acc ? __ldcg(orow + cb + i) : 0.0f);
        }
      }
      if (p.split == 2 && !second) {  // publish this warp's rows of the first half
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.flags + ot, 1u);
      }
      lm::tc_fence_before();
      __syncwarp();
      if (lane == 0) lm::mbar_arrive_cluster(tempty_leader + buf * 8u);
    }
  }

  __syncwarp();
  lm::tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    lm::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
  if (threadIdx.x == 0) {  // every scheduler of this launch is done once all CTAs are here: reset the slot
    __threadfence();
    if (atomicAdd(&p.sched[1], 1u) == gridDim.x - 1) {
      p.sched[0] = 0u;
      p.sched[1] = 0u;
      if (p.split == 2)
        for (int64_t t = 0; t < n_out; ++t) p.flags[t] = 0u;
      __threadfence();
    }
  }
}

template <bool kAMN, bool kBMN>
static cudaError_t launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, GemmParams& p, cudaStream_t stream,
                               int num_sms) {
  const void* fn = (const void*)gemm_tile_kernel<kAMN, kBMN>;
  const size_t smem = gm::smem_bytes();
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int64_t units = dev < 64 ? (int64_t)cached[dev].load(std::memory_order_relaxed) - 1 : -1;
  if (units < 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    units = max_active_clusters(fn, gm::kThreads, smem, 2, num_sms / 2);
    if (dev < 64) cached[dev].store((int)units + 1, std::memory_order_relaxed);
  }
  const int64_t n_tiles = (int64_t)p.n_mt * p.n_nt;
  // split the K loop in two when that fills the last wave better (e.g. dhidden: 320 tiles on 74 clusters, 86 % -> 96 %)
  // and both halves stay long (>= 64 k-blocks)
  p.split = 1;
  if (n_tiles <= kMaxSplitTiles && p.n_kb >= 128) {
    const int64_t U = units;
    auto eff = [U](int64_t t) { const int64_t w = (t + U - 1) / U; return (double)t / (double)(w * U); };
    if (eff(2 * n_tiles) > eff(n_tiles) + 0.05) p.split = 2;  // (a second pass costs a little: only for a clear gain)
  }
  if (units > n_tiles * p.split) units = n_tiles * p.split;
  // half a wave of clusters per group: measured better than a full wave (dweight at 8192 rows 5.99 -> 5.24 ms,
  // 32768 rows 22.3 -> 21.8 ms; dhidden equal or better; 7 stages or a doubled group: no gain)
  p.group_m = (int32_t)(units / (2 * p.n_nt) > 1 ? units / (2 * p.n_nt) : 1);
  unsigned int* slots = nullptr;
  e = cudaGetSymbolAddress((void**)&slots, g_gemm_sched);
  if (e != cudaSuccess) return e;
  unsigned int* flags = nullptr;
  e = cudaGetSymbolAddress((void**)&flags, g_gemm_flags);
  if (e != cudaSuccess) return e;
  const unsigned slot = next_sched_slot(g_gemm_next_slot, g_gemm_next_slot_graph, stream, kGemmSlots);
  p.sched = slots + 2 * slot;
  p.flags = flags + (size_t)slot * kMaxSplitTiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * 2));
  cfg.blockDim = dim3(gm::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_tile_kernel<kAMN, kBMN>, ma, mb, p);
}

// C[M x N] (+)= A B with A(m, k), B(n, k) read from bf16 global memory as described above; row strides in bytes.
cudaError_t gemm_bf16(const void* A, bool a_mn, int64_t a_row_bytes, const void* B, bool b_mn,
                             int64_t b_row_bytes, int64_t M, int32_t N, int32_t K, float* out, int64_t ldo,
                             bool accumulate, cudaStream_t stream, int num_sms) {
  if (M == 0 || N == 0) return cudaSuccess;
  CUtensorMap ma, mb;
  const bool ok_a = a_mn ? make_tensor_map_bf16(&ma, A, (uint64_t)M, (uint64_t)K, (uint64_t)a_row_bytes, 64, 64)
                         : make_tensor_map_bf16(&ma, A, (uint64_t)K, (uint64_t)M, (uint64_t)a_row_bytes, 64, 128);
  const bool ok_b = b_mn ? make_tensor_map_bf16(&mb, B, (uint64_t)N, (uint64_t)K, (uint64_t)b_row_bytes, 64, 64)
                         : make_tensor_map_bf16(&mb, B, (uint64_t)K, (uint64_t)N, (uint64_t)b_row_bytes, 64, 128);
  if (!ok_a || !ok_b) return cudaErrorInvalidValue;
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.n_mt = (int32_t)((M + 255) / 256);
  p.n_nt = (N + gm::kBN - 1) / gm::kBN;
  p.n_kb = (K + gm::kBK - 1) / gm::kBK;
  p.out = out;
  p.ldo = ldo;
  p.accumulate = accumulate ? 1 : 0;
  // an operand small enough to stay in L2 (<= 48 MB, e.g. h of a chunk for dweight) is kept there while the large one
  // streams through with evict_first; with both large, both load with evict_normal (grouped tiles share k-blocks)
  const int64_t a_bytes = M * (int64_t)K * 2, b_bytes = (int64_t)N * K * 2;
  const bool keep_a = a_bytes <= (48ll << 20) && a_bytes < b_bytes;
  const bool keep_b = !keep_a && b_bytes <= (48ll << 20) && b_bytes <= a_bytes;
  p.pol_a = keep_a ? 2 : keep_b ? 1 : 0;
  p.pol_b = keep_b ? 2 : keep_a ? 1 : 0;
  if (a_mn && b_mn) return launch_gemm<true, true>(ma, mb, p, stream, num_sms);
  if (!a_mn && b_mn) return launch_gemm<false, true>(ma, mb, p, stream, num_sms);
  if (!a_mn && !b_mn) return launch_gemm<false, false>(ma, mb, p, stream, num_sms);
  return launch_gemm<true, false>(ma, mb, p, stream, num_sms);
}

cudaError_t tc_lmhead_grads(cudaStream_t stream, int num_sms, const void* weight, const void* hidden_chunk,
                            const void* D, int64_t ld, int64_t rows, int32_t d, int32_t V, float* dhidden_chunk,
                            float* dweight, bool beta_one) {
  // dhidden[rows x d] = D[rows x V] . W[V x d]:  A = D K-major (row stride ld), B = W MN-major ([K = V] x [N = d])
  cudaError_t e = gemm_bf16(D, false, ld * 2, weight, true, (int64_t)d * 2, rows, d, V, dhidden_chunk, d, false,
                            stream, num_sms);
  if (e != cudaSuccess) return e;
  // dweight[V x d] (+)= D^T . h:  A(v, t) = D[t, v] MN-major ([K = rows] x [M = V]), B(j, t) = h[t, j] MN-major
  return gemm_bf16(D, true, ld * 2, hidden_chunk, true, (int64_t)d * 2, V, d, (int32_t)rows, dweight, d, beta_one,
                   stream, num_sms);
}

}  // namespace echo
