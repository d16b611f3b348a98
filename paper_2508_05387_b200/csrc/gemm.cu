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
// filled last wave with a long K loop is avoided by a deterministic S-piece split-K (S <= 8 chosen so that n_tiles * S
// fills whole waves: every piece j of every tile is handed out before any piece j + 1, and piece j's epilogue adds onto
// piece j - 1's stores after a per-tile counter says they are complete -- a fixed fold order, so results do not depend
// on the schedule).
//
// kWide: a unit is the 256 x 512 block of two N-neighbouring tiles, computed by one pair with its two TMEM
// accumulators side by side (512 columns) instead of double-buffering: each k-block loads A once for both tiles (per CTA
// and k-block 48 KB of L2 reads for 2 x 128 x 256 x 64 MACs instead of 2 x 32 KB), and the A operand's DRAM
// re-reads across N halve.  The price: the next unit's MMAs wait for the epilogue.  The epilogue releases accumulator
// 0 first, and the MMA warp runs the next unit's first ring's worth of k-blocks on it alone while accumulator 1 is
// drained (half_rel).  Chosen when N has >= 2 tiles and K >= 128 k-blocks.  (Round 2 also tried 4-CTA clusters
// multicasting A to two pairs: 7-13 % slower; round 3 eight epilogue warps reading a whole accumulator half into
// registers before writing it out: fewer cycles, but a slower training step -- profiles/r3i_epi8_rejected.json.)
#include <cuda.h>
#include <cuda_bf16.h>

#include <stdlib.h>
#include <string.h>

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
template <bool kWide>
struct Smem {
  static constexpr int kSt = kWide ? 4 : kStages;    // ring depth (48 KB stages when wide)
  static constexpr int kNB = kWide ? 2 : 1;          // B tiles per stage
  uint8_t a[kSt][kOpBytes];
  uint8_t b[kSt][kNB][kOpBytes];
  uint8_t ostage[4][2][32 * 128];  // epilogue staging per TMEM lane quadrant, double-buffered: 32 rows x 32 fp32 each,
                                   // SWIZZLE_128B layout
  uint64_t full[kSt], empty[kSt], tfull[2], tempty[2];
  uint64_t tid_full[kTidRing], tid_empty[kTidRing];
  uint32_t tile_id[kTidRing];
  uint32_t tmem_base;
};
// consumers of a tile id: the leader's MMA thread and 4 epilogue warps, the peer's producer thread and 4 epilogue warps
constexpr uint32_t kTidConsumers = 10;
template <bool kWide>
constexpr size_t smem_bytes() { return sizeof(Smem<kWide>) + 1024; }

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
// split-K: per output tile, the number of epilogue-warp completions (8 per finished piece; zeroed at teardown).  Piece j
// of tile t has id j n_out + t, so it is handed out after every piece j - 1 (in-order scheduler: no deadlock -- a
// cluster walks its ids in increasing order, so the piece it waits for is always held by another, earlier cluster)
constexpr int kMaxSplitTiles = 4096;
constexpr int kMaxSplit = 8;
__device__ unsigned int g_gemm_flags[kGemmSlots][kMaxSplitTiles];
static std::atomic<uint32_t> g_gemm_next_slot{0}, g_gemm_next_slot_graph{0};

struct GemmParams {
  int64_t M;
  int32_t N, K, n_mt, n_nt, n_kb, group_m;
  int32_t n_nu;         // N units: N tiles, or (kWide) pairs of N tiles; scheduling unit = (M tile, N unit)
  unsigned int* sched;  // this launch's {tile counter, finished CTAs} (reset by the last CTA)
  unsigned int* flags;  // split-K: this launch's per-output-tile counters
  int32_t split;        // 1..kMaxSplit: K pieces per output tile (id j n_out + t: piece j adds onto piece j - 1)
  int32_t pol_a, pol_b;  // L2 policy per operand: 2 = evict_last (small, re-read by every tile), 1 = evict_first
                         // (streamed past a kept operand), 0 = evict_normal
  float* __restrict__ out;
  int64_t ldo;
  int32_t accumulate;
  int32_t tma_out;  // output 16-B aligned with ldo % 4 == 0: the epilogue writes through map_c (TMA store / L2 add)
  uint32_t ostage_db;  // 1: alternate the two staging boxes per warp; 0: one box (A/B knob ECHO_GEMM_OSTAGE_DB)
  int32_t half_rel;    // kWide: the epilogue releases the two 256-column accumulators one by one (ECHO_GEMM_HALFREL)
};

template <bool kAMN, bool kBMN, bool kWide>
__global__ void __launch_bounds__(gm::kThreads, 1)
    gemm_tile_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ CUtensorMap map_c, const GemmParams p) {
  using namespace gm;
  using S = Smem<kWide>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  S& sm = *reinterpret_cast<S*>(smem_raw + (((raw + 1023u) & ~1023u) - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_units = (int64_t)p.n_mt * p.n_nu, n_tiles = n_units * p.split;
  // k-block range of piece j: [j n_kb / S, (j + 1) n_kb / S)
  auto kb_begin = [&](int32_t j) { return (int32_t)(((int64_t)j * p.n_kb) / p.split); };
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  constexpr int kUnitN = kWide ? 2 * kBN : kBN;  // output columns of a unit
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
    else lm::mbar_arrive_cluster(mapa(smem_u32(&sm.tid_empty[r]), 0));
  };
  // accumulator of the tc-th unit: double-buffered, or (kWide) both 256-column halves of TMEM, one unit at a time
  auto acc_buf = [&](uint32_t tc) -> uint32_t { return kWide ? 0u : (tc & 1u); };
  auto acc_phase = [&](uint32_t tc) -> uint32_t { return kWide ? (tc & 1u) : ((tc >> 1) & 1u); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::kSt; ++s) {
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
    if (p.tma_out) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
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
        if (leader) {  // the scheduler: grab the next unit, publish it to this CTA and the peer
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
        int32_t mt, nu;
        const int32_t piece = (int32_t)(u / n_units);  // split-K piece
        tile_coords(u - (int64_t)piece * n_units, p.n_mt, p.n_nu, p.group_m, mt, nu);
        const int32_t m_row = mt * 256 + (int32_t)rank * kBM, n_row = nu * kUnitN + (int32_t)rank * 128;
        const int32_t kb0 = kb_begin(piece), kb1 = kb_begin(piece + 1);
        for (int32_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&sm.empty[stage]), phase ^ 1u);
          const uint32_t bar = mapa(smem_u32(&sm.full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(smem_u32(&sm.full[stage]), 2 * (1 + S::kNB) * kOpBytes);
          load_op<kAMN>(smem_u32(sm.a[stage]), &map_a, m_row, kb * kBK, bar, pol_a);
#pragma unroll
          for (int j = 0; j < S::kNB; ++j)  // kWide: the second N tile's half, 256 columns further
            load_op<kBMN>(smem_u32(sm.b[stage][j]), &map_b, n_row + j * kBN, kb * kBK, bar, pol_b);
          if (++stage == S::kSt) {
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
        const uint32_t buf = acc_buf(tc), aph = acc_phase(tc);
        mbar_wait_cluster(smem_u32(&sm.tempty[buf]), aph ^ 1u);
        lm::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * kBN;
        const int32_t piece = (int32_t)(u / n_units);
        const int32_t kb0 = kb_begin(piece), kb1 = kb_begin(piece + 1);
        int32_t kb_first = kb0;
        if (kWide && p.half_rel) {
          // The epilogue frees the first accumulator half-way through its read-out (tempty[0]) and the second at the
          // end (tempty[1]): run the first ring's worth of k-blocks on accumulator 0 alone while accumulator 1 is
          // still being drained, then the same stages again on accumulator 1, releasing them.
          const int32_t nhead = min(S::kSt, kb1 - kb0);
          uint32_t st = stage, ph = phase;
          for (int32_t i = 0; i < nhead; ++i) {
            mbar_wait_cluster(smem_u32(&sm.full[st]), ph);
            lm::tc_fence_after();
            const uint32_t a0 = smem_u32(sm.a[st]);
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
              lm::umma_f16<true>(d_tmem, op_desc<kAMN>(a0, k), op_desc<kBMN>(smem_u32(sm.b[st][0]), k),
                                 idesc<kAMN, kBMN>(), (i > 0 || k > 0) ? 1u : 0u);
            if (++st == S::kSt) {
              st = 0;
              ph ^= 1u;
            }
          }
          mbar_wait_cluster(smem_u32(&sm.tempty[1]), aph ^ 1u);
          lm::tc_fence_after();
          for (int32_t i = 0; i < nhead; ++i) {
            const uint32_t a0 = smem_u32(sm.a[stage]);
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
              lm::umma_f16<true>(d_tmem + kBN, op_desc<kAMN>(a0, k), op_desc<kBMN>(smem_u32(sm.b[stage][S::kNB - 1]), k),
                                 idesc<kAMN, kBMN>(), (i > 0 || k > 0) ? 1u : 0u);
            lm::umma_commit<true>(smem_u32(&sm.empty[stage]));
            if (++stage == S::kSt) {
              stage = 0;
              phase ^= 1u;
            }
          }
          kb_first = kb0 + nhead;
        }
        for (int32_t kb = kb_first; kb < kb1; ++kb) {
          mbar_wait_cluster(smem_u32(&sm.full[stage]), phase);
          lm::tc_fence_after();
          const uint32_t a0 = smem_u32(sm.a[stage]);
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k) {
#pragma unroll
            for (int j = 0; j < S::kNB; ++j)
              lm::umma_f16<true>(d_tmem + j * kBN, op_desc<kAMN>(a0, k), op_desc<kBMN>(smem_u32(sm.b[stage][j]), k),
                                 idesc<kAMN, kBMN>(), (kb > kb0 || k > 0) ? 1u : 0u);
          }
          lm::umma_commit<true>(smem_u32(&sm.empty[stage]));  // the stage is free once these MMAs have read it
          if (++stage == S::kSt) {
            stage = 0;
            phase ^= 1u;
          }
        }
        lm::umma_commit<true>(smem_u32(&sm.tfull[buf]));
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5 = TMEM lane quadrants)
    // thread = output row (TMEM lane), 32 fp32 columns per tcgen05.ld.  TMA path: the warp's 32 x 32 block goes to
    // its shared-memory staging box (16-byte granule j of row r at j ^ (r & 7): the SWIZZLE_128B layout) and one lane
    // writes it with a tensor-map store, or with an add performed in L2 (cp.reduce.async.bulk .add) when
    // accumulating -- no global loads, full-line writes, a few instructions per 1024 outputs.
    const int quad = warp & 3;
    uint32_t tc = 0;
    const uint32_t tempty_leader = mapa(smem_u32(&sm.tempty[0]), 0);
    const bool vec_ok = (p.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
    const uint32_t ostage0 = smem_u32(sm.ostage[quad][0]);
    uint32_t nstaged = 0;  // boxes this warp has handed to the TMA unit (picks the staging buffer)
    for (;; ++tc) {
      const int64_t u = next_tile_warp(tc);
      __syncwarp();
      if (lane == 0) release_tile(tc);
      if (u >= n_tiles) break;
      int32_t mt, nu;
      const int32_t piece = (int32_t)(u / n_units);
      const int64_t ot = u - (int64_t)piece * n_units;  // output unit (split-K counter index)
      tile_coords(ot, p.n_mt, p.n_nu, p.group_m, mt, nu);
      const uint32_t buf = acc_buf(tc), aph = acc_phase(tc);
      const int64_t row0 = (int64_t)mt * 256 + (int64_t)rank * kBM + quad * 32;  // this warp's 32 output rows
      const int64_t row = row0 + lane;
      const bool row_ok = row < p.M;
      float* orow = p.out + (row_ok ? row : 0) * p.ldo;
      // split-K: piece j > 0 adds onto piece j - 1's stores (fixed order: deterministic)
      const bool second = piece > 0;
      const bool acc = p.accumulate || second;
      mbar_wait_cluster_warp(smem_u32(&sm.tfull[buf]), aph, lane);
      lm::tc_fence_after();
      if (second) {
        if (lane == 0) {
          uint32_t v;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.flags + ot) : "memory");
            if (v >= 8u * (uint32_t)piece) break;
            __nanosleep(256);
          }
          if (p.tma_out) lm::fence_proxy_async_all();  // the L2 adds below are ordered after the acquire
        }
        __syncwarp();
        __threadfence();
      }
      // kWide with half_rel: accumulator 0 (columns 0-255) is released after its 8 chunks, accumulator 1 after the rest
      const int n_halves = (kWide && p.half_rel) ? 2 : 1, ch_per = (kUnitN / 32) / n_halves;
      for (int h = 0; h < n_halves; ++h) {
#pragma unroll 1
        for (int ch = h * ch_per; ch < (h + 1) * ch_per; ++ch) {
          const int32_t cb = nu * kUnitN + ch * 32;
          if (cb >= p.N) break;  // warp-uniform
          uint32_t r[32];
          lm::tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + buf * kBN + ch * 32, r);
          if (p.tma_out) {
            if (row0 >= p.M) continue;  // warp-uniform: the whole 32-row block is past the end
            // the buffer's previous box (two boxes ago) has been read by its TMA; the other one may still be in flight
            const uint32_t ostage = ostage0 + (nstaged & p.ostage_db) * (32u * 128u);
            if (lane == 0) {
              if (p.ostage_db) lm::bulk_wait_read1();
              else lm::bulk_wait_read0();
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              sts_v4(ostage + (uint32_t)lane * 128u + ((uint32_t)(j ^ (lane & 7)) << 4),
                     make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]));
            lm::fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) {
              if (acc) lm::tma_reduce_add_2d(&map_c, ostage, cb, (int32_t)row0);
              else lm::tma_store_2d(&map_c, ostage, cb, (int32_t)row0);
              lm::bulk_commit();
            }
            ++nstaged;
            continue;
          }
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
        // the accumulator (half) has been read: release it to the MMA of the tile after next (kWide: the next unit)
        lm::tc_fence_before();
        __syncwarp();
        if (lane == 0) lm::mbar_arrive_cluster(tempty_leader + (n_halves == 2 ? (uint32_t)h : buf) * 8u);
      }
      if (piece + 1 < p.split) {  // publish this warp's rows of piece j (complete in global memory)
        if (p.tma_out && lane == 0) {
          lm::bulk_wait0();
          lm::fence_proxy_async_all();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.flags + ot, 1u);
      }
    }
    if (p.tma_out && lane == 0) lm::bulk_wait0();  // staging boxes read and writes done before the CTA retires
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
      if (p.split > 1)
        for (int64_t t = 0; t < n_units; ++t) p.flags[t] = 0u;
      __threadfence();
    }
  }
}

template <bool kAMN, bool kBMN, bool kWide>
static cudaError_t launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, GemmParams& p,
                               cudaStream_t stream, int num_sms) {
  const void* fn = (const void*)gemm_tile_kernel<kAMN, kBMN, kWide>;
  const size_t smem = gm::smem_bytes<kWide>();
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int64_t units = dev < 64 ? (int64_t)cached[dev].load(std::memory_order_relaxed) - 1 : -1;  // resident clusters
  if (units < 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    units = max_active_clusters(fn, gm::kThreads, smem, 2, num_sms / 2);
    if (dev < 64) cached[dev].store((int)units + 1, std::memory_order_relaxed);
  }
  p.n_nu = kWide ? (p.n_nt + 1) / 2 : p.n_nt;
  const int64_t n_work = (int64_t)p.n_mt * p.n_nu;
  // split the K loop into S pieces when that fills the last wave better (dhidden at 8192 rows: 320 tiles on 74
  // clusters fill 86 % of 5 waves; S = 3 fills 99.8 % of 13) and every piece stays long (>= 64 k-blocks).  Each extra
  // piece costs one add-onto-the-output epilogue pass, hence the small per-piece penalty.
  p.split = 1;
  if (n_work <= kMaxSplitTiles) {
    const int64_t U = units;
    auto eff = [U](int64_t t) { const int64_t w = (t + U - 1) / U; return (double)t / (double)(w * U); };
    double best = eff(n_work);
    for (int32_t sp = 2; sp <= kMaxSplit && p.n_kb / sp >= 64; ++sp) {
      const double e2 = eff(sp * n_work) - 0.01 * (sp - 1);
      if (e2 > best + 0.02) {
        best = e2;
        p.split = sp;
      }
    }
  }
  if (const char* env = getenv("ECHO_GEMM_SPLIT")) {  // A/B knob: force S (K pieces of >= 64 k-blocks)
    const int32_t sp = atoi(env);
    if (sp >= 1 && sp <= kMaxSplit && p.n_kb / sp >= 64 && n_work <= kMaxSplitTiles) p.split = sp;
  }
  if (units > n_work * p.split) units = n_work * p.split;
  // raster group: half a wave of clusters (measured better than a full wave at d = 2560: dweight at 8192 rows 5.99 ->
  // 5.24 ms), but 16 M tiles once there are >= 16 N units -- the tiles in flight then span ~16 M x 4.6 N tiles instead
  // of ~4 x 20, cutting the DRAM re-reads of the N-side operand (interleaved A/B at d = 5120, 8192 rows: dhidden
  // 11.81 -> 10.66 ms, dweight 11.28 -> 10.51 ms; profiles/r2i_ab_knobs.jsonl)
  p.group_m = (int32_t)(units / (2 * p.n_nu) > 1 ? units / (2 * p.n_nu) : 1);
  if (p.n_nu >= 16) p.group_m = 16;
  // 256 x 512 units with 8-15 N units (d = 4096-7680): 8 M tiles per group (the chunked f2 step at d = 5120: 118.6-119.0
  // vs 120.4-121.5 ms with the half-wave group of 3, 121.4 with 16; profiles/r3b_f2step_knobs.jsonl)
  else if (kWide && p.n_nu >= 8) p.group_m = 8;
  p.half_rel = 1;
  if (const char* env = getenv("ECHO_GEMM_HALFREL")) p.half_rel = atoi(env) != 0;  // A/B knob
  p.ostage_db = 1;
  if (const char* env = getenv("ECHO_GEMM_OSTAGE_DB")) p.ostage_db = atoi(env) != 0;  // A/B knob
  if (const char* env = getenv("ECHO_GEMM_GROUP")) p.group_m = atoi(env) > 0 ? atoi(env) : p.group_m;  // A/B knob
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
  return cudaLaunchKernelEx(&cfg, gemm_tile_kernel<kAMN, kBMN, kWide>, ma, mb, mc, p);
}

template <bool kWide>
static cudaError_t launch_majors(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                                 const CUtensorMap& mc, GemmParams& p, cudaStream_t stream, int num_sms) {
  if (a_mn && b_mn) return launch_gemm<true, true, kWide>(ma, mb, mc, p, stream, num_sms);
  if (!a_mn && b_mn) return launch_gemm<false, true, kWide>(ma, mb, mc, p, stream, num_sms);
  if (!a_mn && !b_mn) return launch_gemm<false, false, kWide>(ma, mb, mc, p, stream, num_sms);
  return launch_gemm<true, false, kWide>(ma, mb, mc, p, stream, num_sms);
}

// C[M x N] (+)= A B with A(m, k), B(n, k) read from bf16 global memory as described above; row strides in bytes.
cudaError_t gemm_bf16(const void* A, bool a_mn, int64_t a_row_bytes, const void* B, bool b_mn,
                             int64_t b_row_bytes, int64_t M, int32_t N, int32_t K, float* out, int64_t ldo,
                             bool accumulate, cudaStream_t stream, int num_sms) {
  if (M == 0 || N == 0) return cudaSuccess;
  // 256 x 512 units (two accumulators sharing A) whenever there are N tiles to pair and the K loop is not short: every A
  // k-block feeds two tiles, so A's L2 reads halve and its DRAM re-reads across N too (ncu, dhidden 8192 x 5120 x
  // 151936: 12.7 vs 25.6 GB of DRAM reads, 2.43 vs 3.32 G L2 sectors, 1.34 vs 1.24 GHz, 8.1 vs 9.3 ms), and the
  // power-capped clock rises.  Inside the chunked f2 step (tools/prof_f2_step.py, d = 5120, 8192-row chunks,
  // profiles/r3a_f2step_wide.jsonl) the step's four GEMM-heavy stages take 122.0 ms instead of 134.0 (cuBLAS for
  // the two backward products: 117.3).  Only back-to-back launches on warm, identical inputs favour 256 x 256 units
  // (profiles/r2z_ab_wide_sus.jsonl).  ECHO_GEMM_WIDE=0/1 overrides, for A/B.
  const int32_t n_kb = (K + gm::kBK - 1) / gm::kBK, n_nt = (N + gm::kBN - 1) / gm::kBN;
  bool wide = n_nt >= 2 && n_kb >= 128;
  if (const char* env = getenv("ECHO_GEMM_WIDE")) wide = atoi(env) != 0 && n_nt >= 2;
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
  // output through a tensor map (box 32 columns x 32 rows of fp32, SWIZZLE_128B) when its layout allows
  // (N % 4: a tensor-map store writes whole 16-byte granules, so a ragged last granule would spill past column N)
  CUtensorMap mc_map;
  memset(&mc_map, 0, sizeof(mc_map));
  p.tma_out = (ldo % 4 == 0 && N % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
               make_tensor_map_f32(&mc_map, out, (uint64_t)N, (uint64_t)M, (uint64_t)ldo * 4, 32, 32))
                  ? 1
                  : 0;
  // L2 policy: the smaller operand loads with evict_last, the other with evict_normal.  Both are re-read by the units
  // in flight (A by the N units of its M tile, B by the M tiles of the group), so neither is streamed with
  // evict_first.  Sustained at the 1000 W power cap (tools/power_probe.py, profiles/r3t_power_pol.jsonl,
  // r3u_power_pol.jsonl): dweight at d = 2560 5.00 instead of 5.28 ms (the former rule: h evict_last, D
  // evict_first), at d = 5120 10.04 instead of 10.20 (former: both normal), dhidden at d = 5120 9.83 instead of 10.00;
  // evict_first on D costs 10 %.
  const int64_t a_bytes = M * (int64_t)K * 2, b_bytes = (int64_t)N * K * 2;
  p.pol_a = a_bytes < b_bytes ? 2 : 0;
  p.pol_b = a_bytes < b_bytes ? 0 : 2;
  if (const char* env = getenv("ECHO_GEMM_POL_A")) p.pol_a = atoi(env);  // A/B knobs: 0 normal, 1 first, 2 last
  if (const char* env = getenv("ECHO_GEMM_POL_B")) p.pol_b = atoi(env);
  return wide ? launch_majors<true>(a_mn, b_mn, ma, mb, mc_map, p, stream, num_sms)
              : launch_majors<false>(a_mn, b_mn, ma, mb, mc_map, p, stream, num_sms);
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
