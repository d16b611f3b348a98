// policy_loss_quad.cu -- ECHO_ALGO_QUAD_REG / _EXACT: the B200 design of the fused (3)+(4)+(5) kernel.
//
// One logits row (V ~ 152k bf16 = 297 KB) is owned by a thread-block cluster of C::kCtas = 4 CTAs; CTA r holds
// the quarter [r q, (r+1) q) of the row (q = ceil(V/4) rounded to 8) in REGISTERS: 8 warps x 32 threads x
// 19 vectors of 16 B = 76 registers per thread.  Two such CTAs share an SM (registers 2 x 256 x 128 = 64 K,
// shared memory 2 x 112 KB), so every SM always has two rows in flight: while one CTA waits on its cluster
// merge or drains its stores, the other keeps the MUFU / FMA pipes busy.  The persistent grid (as many 4-CTA
// clusters as fit: 71 on a B200) takes rows in order from a global counter (rank 0 of each cluster grabs and
// broadcasts them), so all clusters stream one compact window of consecutive rows; HBM sees exactly one read
// and one write per logit.
//
// Per CTA and row:
//   stage    1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx) stream the quarter-row through a
//            28 x 4 KB shared-memory ring, one barrier per row; warp 1 refills the slots of row it as soon as the
//            CTA barrier after pass 1b shows they have been copied into registers, so row it+1 and the head of
//            row it+2 are always in flight
//   pass 1a  ring -> registers, exact bf16x2 running max m_t; thread 0 reads z_a from the ring
//   pass 1b  e = 2^((z - m_t) log2e) (MUFU), s_t = sum e (FADD2); kStoreExp: registers <- e as fp16
//   merge    (m_t, s_t) -> warp (xor shuffles) -> CTA (warp 0) -> cluster: each CTA st.async's its
//            {m, s, z_a} into slot [rank] of every peer's shared memory, completing 16 tx-bytes on the peer's
//            mbarrier; all CTAs merge the 4 partials in rank order -> identical lse bits everywhere
//   epilogue lse, logp, rho, clip, KL, c_t (fp32), rank 0 writes the per-token outputs
//   pass 2   d = e k_t (k_t = -c_t 2^((m_t - lse) log2e), FMUL2)  or, exact, d = -c_t 2^((z - lse) log2e);
//            bf16 RNE, 16-byte stores in place; the action column gets c_t (1 - p_a) from the fp32 epilogue
// Determinism: the reduction tree depends only on V and the tile constants, never on the grid, the rank or
// which cluster a row is scheduled on.
#include <cuda_bf16.h>

#include <stdlib.h>

#include <atomic>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

// Tile configurations: a row is split across kCtas CTAs of kWarps warps; 16 warps per SM (4 per SM
// sub-partition) leaves 128 registers per thread, of which 76 hold the thread's 19 vectors of the row.
//   QCfg<4, 8>: 4-CTA cluster, 2 CTAs (2 rows) per SM  -- ECHO_ALGO_QUAD_REG
//   QCfg<8, 4>: 8-CTA cluster, 4 CTAs (4 rows) per SM  -- ECHO_ALGO_OCT_REG
//   QCfg<16, 4>: 16-CTA cluster, 4 CTAs per SM          -- ECHO_ALGO_HEX_REG (vocabularies up to 311296)
//   QCfg<16, 4, false, 10, 8>: logp mode only -- 16-CTA cluster, 8 CTAs per SM (32 warps), 10 vectors per thread
template <int kCtas_, int kWarps_, bool kF32_ = false, int kRegChunks_ = 19, int kCtasPerSm_ = 16 / kWarps_>
struct QCfg {
  static constexpr int kCtas = kCtas_;                  // CTAs per row (cluster size)
  static constexpr int kWarps = kWarps_;                // all warps compute; warp 0 also issues the TMA loads
  static constexpr bool kF32 = kF32_;                   // fp32 logits (else bf16)
  static constexpr int kElemBytes = kF32 ? 4 : 2;
  static constexpr int kVecElems = 16 / kElemBytes;     // logits per 16-byte vector
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kChunk = kThreads * 16;          // one 16-byte vector per thread
  static constexpr int kChunkElems = kChunk / kElemBytes;
  static constexpr int kCtasPerSm = kCtasPerSm_;
  // staging ring slots (~1.5 slices; fills the SM's shared memory)
  static constexpr int kRing = kCtasPerSm == 2 ? 28 : kCtasPerSm == 4 ? 27 : 13;
  static constexpr int kRegChunks = kRegChunks_;        // V <= kCtas * kRegChunks * kChunkElems (155648 for 8 x 19)
};
constexpr int kQBar = 1;                                // named barrier id

// per-row metadata, staged in shared memory by thread 0 with cp.async one row ahead (keeps it out of registers)
struct MetaSm {
  int32_t a, slot;
  float old, ref, adv, w;
};

template <class C>
struct __align__(128) QuadSmem {
  uint8_t ring[C::kRing][C::kChunk];
  uint64_t full[4];      // per row (it % 4): all chunks of the row landed (one complete_tx per chunk)

  uint64_t xbar[2];
  uint4 xbuf[2][C::kCtas];  // cluster partials {m, s, z_a, -} per row parity and source rank
  float red_m[2][C::kWarps];  // per row parity: in logp mode the next row's warps run ahead of warp 0's merge
  float red_s[2][C::kWarps];
  float red_t[2][C::kWarps];  // kModeEntropy: sum z e^{z - m} per warp
  float za;
  MetaSm meta[2];        // rows of iterations it (it & 1) and it+1
  float coef;
  float lse;
  float da;
  float ent_k;           // kModeEntropy: eta s w (H - lse) - c_t
  float ent_e;           // kModeEntropy: eta s w
  uint64_t rowbar[4];    // row table: iteration k's row lands in rowtab[k % 4] (st.async from rank 0)
  int64_t rowtab[4];
};

// Dynamic row scheduling.  Rank 0 of each cluster takes rows from a global counter in order and broadcasts them
// to the cluster's row tables 3 iterations ahead, so all clusters work inside one compact window of consecutive
// rows.  With a static stride (row = cluster + it * n_clusters) the clusters drift apart and the in-flight
// addresses spread over hundreds of MB; the compact window sustains ~9% more HBM bandwidth on the same access
// pattern (tools/membench.cu: ring_read_write 3.16 -> 2.91 ms).  One {next row, CTAs done} pair per launch slot;
// a launch takes the next slot round-robin and its last CTA resets the pair, so no memset is needed.
constexpr int kSchedSlots = 256;
__device__ unsigned long long g_row_sched[kSchedSlots][2];
static std::atomic<uint32_t> g_next_sched_slot{0}, g_next_sched_slot_graph{0};  // shared by every tile / mode
constexpr int kMaxDevices = 64;
constexpr int kRowAhead = 3;
  // rows are broadcast this many iterations ahead (<= 4: the table depth)

struct QuadGeom {
  int32_t q;               // slice width: rank r owns [r q, min((r+1) q, V))
  int32_t c0, c1;          // this CTA's columns [c0, c1)
  uint32_t slice_bytes;    // bytes loaded per row (c1 rounded up to 8 columns)
  int nchunks;             // ring chunks per row
};

template <class C>
ECHO_DEVINL QuadGeom quad_geom(int32_t V, uint32_t rank) {
  QuadGeom g;
  constexpr int32_t E = C::kVecElems;
  const int32_t q = ((V + C::kCtas - 1) / C::kCtas + E - 1) & ~(E - 1);
  g.q = q;
  // slices start on vector (16-byte) boundaries; a rank past the end gets an empty slice [V_E, V_E)
  const int32_t vE = (V + E - 1) & ~(E - 1);
  g.c0 = min((int32_t)rank * q, vE);
  g.c1 = max(min((int32_t)(rank + 1) * q, V), g.c0);
  const int32_t c1r = (g.c1 + E - 1) & ~(E - 1);
  g.slice_bytes = (uint32_t)(c1r - g.c0) * (uint32_t)C::kElemBytes;
  g.nchunks = (int)((g.slice_bytes + C::kChunk - 1) / C::kChunk);
  return g;
}

// Issue chunks [from, to) of this CTA's chunk stream (iteration j = q / nchunks, chunk q % nchunks) into ring slot
// q % kRing, one lane per chunk; rows[j - it0] is iteration j's row (j - it0 in {0, 1, 2}).  The lane that issues
// an iteration's chunk 0 arms that iteration's barrier with the slice byte count (tx may transiently go negative;
// the phase cannot complete before the arrive).
template <class C>
ECHO_DEVINL void quad_issue_chunks(const LossParams& p, const QuadGeom& g, uint32_t from, uint32_t to, int lane,
                                   uint32_t full0, uint32_t ring0, uint64_t pol, uint32_t it0, int64_t row0,
                                   int64_t row1, int64_t row2) {
  for (uint32_t q = from + (uint32_t)lane; q < to; q += 32) {
    const uint32_t j = q / (uint32_t)g.nchunks, c = q % (uint32_t)g.nchunks;
    const uint32_t bar = full0 + 8 * (j & 3u);
    if (c == 0) mbar_arrive_expect_tx(bar, g.slice_bytes);
    const int64_t row = j == it0 ? row0 : j == it0 + 1 ? row1 : row2;
    const uint8_t* src = p.logits + row * p.ld_bytes + (int64_t)g.c0 * C::kElemBytes + (int64_t)c * C::kChunk;
    const uint32_t nb = min((uint32_t)C::kChunk, g.slice_bytes - c * C::kChunk);
    bulk_g2s(ring0 + (q % C::kRing) * C::kChunk, src, nb, bar, pol);
  }
}

// kMode: kModeExact (gradient, exp recomputed in pass 2), kModeCache (gradient, exp kept as fp16 between the
// passes), kModeLogp (forward only: log-probs and lse, the logits are not written -- SURVEY.md §8.6 f1).
// kModeEntropy: kModeExact plus the entropy bonus (f4): pass 1 also accumulates t = sum z e^{z - m}, the cluster
// merge carries (m, s, t), H = lse - t / s, and pass 2 adds the entropy gradient p (log p + H) eta s w.
enum { kModeExact = 0, kModeCache = 1, kModeLogp = 2, kModeEntropy = 3 };

template <class C, int kMode>
__global__ void __cluster_dims__(C::kCtas, 1, 1) __launch_bounds__(C::kThreads, C::kCtasPerSm)
    policy_loss_quad_kernel(const LossParams p) {
  constexpr bool kStoreExp = kMode == kModeCache;
  constexpr bool kGrad = kMode != kModeLogp;
  constexpr bool kEnt = kMode == kModeEntropy;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  QuadSmem<C>& sm = *reinterpret_cast<QuadSmem<C>*>(smem_raw);
  const uint32_t rank = cluster_ctarank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t V = p.V;
  const QuadGeom g = quad_geom<C>(V, rank);
  const int nchunks = g.nchunks;
  const int32_t c0 = g.c0, c1 = g.c1;
  const uint32_t full0 = smem_u32(&sm.full[0]), ring0 = smem_u32(&sm.ring[0][0]);
  const int64_t n_rows = p.n_rows;
  unsigned long long* const sched = g_row_sched[p.sched_slot];
  const uint32_t rowbar0 = smem_u32(&sm.rowbar[0]);

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(rowbar0 + 8 * i, 1);
      mbar_arrive_expect_tx(rowbar0 + 8 * i, 8);  // phase i: row of iteration i
    }
    mbar_init(smem_u32(&sm.xbar[0]), 1);
    mbar_init(smem_u32(&sm.xbar[1]), 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();

  // iteration k's row (waits for rank 0's broadcast)
  auto row_of = [&](uint32_t k) -> int64_t {
    mbar_wait_cluster(rowbar0 + 8 * (k & 3u), (k >> 2) & 1u);
    return *reinterpret_cast<volatile int64_t*>(&sm.rowtab[k & 3u]);
  };
  auto broadcast = [&](uint32_t k, unsigned long long r) {
#pragma unroll
    for (int q = 0; q < C::kCtas; ++q)
      st_async_b64(mapa(smem_u32(&sm.rowtab[k & 3u]), q), r, mapa(rowbar0 + 8 * (k & 3u), q));
  };
  // rank 0's warp 1 lane 0 runs the scheduler: rows of iterations 0..2 now, then one row per iteration
  // (the next grab is issued one iteration before it is broadcast, so its latency stays off the critical path)
  const bool sched_thread = rank == 0 && tid == 32;
  bool sched_done = true;
  unsigned long long grabbed = 0;
  if (sched_thread) {
    const unsigned long long r0 = atomicAdd(&sched[0], (unsigned long long)kRowAhead);
    sched_done = false;
    for (int k = 0; k < kRowAhead && !sched_done; ++k) {
      const unsigned long long r = r0 + k < (unsigned long long)n_rows ? r0 + k : (unsigned long long)n_rows;
      broadcast(k, r);
      sched_done = r >= (unsigned long long)n_rows;
    }
    if (!sched_done) grabbed = atomicAdd(&sched[0], 1ull);
  }

  // warp 1 streams the rows: the ring holds ~1.4 rows, so row it+1 and the head of row it+2 are in flight while
  // row it is reduced; slots are refilled once the CTA barrier after pass 1b shows row it has been copied out
  uint32_t issued = 0;
  if (warp == 1 && nchunks > 0) {
    const int64_t r0 = row_of(0);
    const int64_t r1 = r0 < n_rows ? row_of(1) : n_rows;
    const int64_t r2 = r1 < n_rows ? row_of(2) : n_rows;
    const uint32_t rows_ok = r0 >= n_rows ? 0u : r1 >= n_rows ? 1u : r2 >= n_rows ? 2u : 3u;
    issued = min((uint32_t)C::kRing, rows_ok * (uint32_t)nchunks);
    quad_issue_chunks<C>(p, g, 0, issued, lane, full0, ring0, policy_evict_normal(), 0, r0, r1, r2);
  }

  const float gscale = kGrad ? base_scale(p) : 0.0f;
  constexpr int32_t E = C::kVecElems;
  constexpr uint32_t kNegInf2 = C::kF32 ? 0xFF800000u : kBf16NegInf2;  // -inf in every lane of a word
  const int32_t col_t = c0 + tid * E;
  const bool last_valid = (uint32_t)(nchunks - 1) * C::kChunk + (uint32_t)tid * 16u < g.slice_bytes;
  const bool has_tail = (c1 & (E - 1)) && (c1 & ~(E - 1)) >= col_t && ((c1 & ~(E - 1)) - col_t) % C::kChunkElems == 0;
  const int nstore = nchunks - (last_valid ? 0 : 1) - (has_tail ? 1 : 0);
  const uint64_t l2e2 = f2(kLog2e, kLog2e);
  const uint32_t my_off = (uint32_t)tid * 16u;

  // Per-row metadata is staged one row ahead so its global-load latency never sits on the critical path.
  // Thread 0, per iteration it: group C(it) = the dependent advantage load of row it (its slot landed with A(it)),
  // then group A(it+1) = action, old, ref, weight, slot / per-token advantage of row it+1.  A(it+1) is complete
  // before barrier 2 of iteration it (which publishes the action to every thread), C(it) before the epilogue.
  auto stage_meta = [&](int64_t r, uint32_t k) {
    MetaSm& m = sm.meta[k & 1u];
    cp_async4(smem_u32(&m.a), p.tok_action + r);
    if constexpr (kGrad) {
      cp_async4(smem_u32(&m.old), p.tok_old + r);
      if (p.kl_coef > 0.0f) cp_async4(smem_u32(&m.ref), p.tok_ref + r);
      else m.ref = 0.0f;
      if (p.tok_weight) cp_async4(smem_u32(&m.w), p.tok_weight + r);
      else m.w = 1.0f;
      if (p.tok_adv) cp_async4(smem_u32(&m.adv), p.tok_adv + r);
      else cp_async4(smem_u32(&m.slot), p.tok_slot + r);
    }
  };
  int64_t row_next = row_of(0);
  if (tid == 0 && row_next < n_rows) {
    stage_meta(row_next, 0);
    cp_async_commit();
    cp_async_wait<0>();
  }
  named_bar_sync(kQBar, C::kThreads);
  // Cluster merge of row k (lane 0 of warp 0): wait for the kCtas partials, merge them in rank order -- max first,
  // then the rescaled sums (the exps are independent) -- and run the row's epilogue.  The partials are re-read from
  // shared memory rather than held (4 words per rank would cost registers).
  auto finish = [&](uint32_t k, int64_t row_k, int32_t a_k) {
    const uint32_t par = k & 1u;
    mbar_wait_cluster(smem_u32(&sm.xbar[par]), (k >> 1) & 1u);
    ECHO_TRACE_MARK(p, k, 7);
    float mm = -INFINITY;
#pragma unroll
    for (int r = 0; r < C::kCtas; ++r) mm = fmaxf(mm, __uint_as_float(sm.xbuf[par][r].x));
    float ss = 0.0f, tt = 0.0f;
#pragma unroll
    for (int r = 0; r < C::kCtas; ++r) {
      const float mr = __uint_as_float(sm.xbuf[par][r].x), sr = __uint_as_float(sm.xbuf[par][r].y);
      const float f = (mr == -INFINITY) ? 0.0f : ex2((mr - mm) * kLog2e);
      ss += sr * f;
      if (kEnt) tt += __uint_as_float(sm.xbuf[par][r].z) * f;
    }
    const float lse = mm + logf(ss);
    const float za = (a_k < 0 || a_k >= V) ? NAN : __uint_as_float(sm.xbuf[par][a_k / g.q].w);
    if constexpr (kGrad) {
      cp_async_wait<1>();  // C(k) landed
      const MetaSm& m = sm.meta[k & 1u];
      const float H = kEnt ? lse - tt / ss : 0.0f;  // -sum p log p = lse - sum p z
      const RowScalars r = row_epilogue(lse, za, m.old, m.ref, m.adv, loss_opts(p), gscale * m.w, H);
      if (rank == 0) {
        p.tok_logp[row_k] = r.logp;
        p.tok_loss[row_k] = r.loss;
        p.tok_flags[row_k] = r.flags;
        if (kEnt && p.tok_entropy) p.tok_entropy[row_k] = H;
      }
      const float pa = ex2(fmaf(za, kLog2e, -lse * kLog2e));
      sm.coef = r.coef;
      sm.lse = lse;
      sm.da = fmaf(-r.coef, pa, r.coef);
      if (kEnt) {
        sm.ent_e = r.ecoef;
        sm.ent_k = fmaf(r.ecoef, H - lse, -r.coef);
        sm.da = fmaf(r.ecoef * pa, za - lse + H, sm.da);  // c (1 - p_a) + e p_a (log p_a + H)
      }
    } else if (rank == 0) {
      const float logp = za - lse;
      p.tok_logp[row_k] = logp;
      if (p.tok_lse) p.tok_lse[row_k] = lse;
      if (p.tok_flags) p.tok_flags[row_k] = (isfinite(lse) && isfinite(logp)) ? 0 : ECHO_FLAG_NONFINITE;
    }
  };
  for (uint32_t it = 0;; ++it) {
    const int64_t row = row_next;
    if (row >= n_rows) break;
    const int32_t a = sm.meta[it & 1u].a;
    row_next = row_of(it + 1);
    if (tid == 0) {
      if (kGrad && !p.tok_adv) cp_async4(smem_u32(&sm.meta[it & 1u].adv), p.adv_slot + sm.meta[it & 1u].slot);
      cp_async_commit();
      if (row_next < n_rows) stage_meta(row_next, it + 1);
      cp_async_commit();
    }

    ECHO_TRACE_MARK(p, it, 0);
    // ---- pass 1a: one wait for the whole row, then ring -> registers
    uint4 v[C::kRegChunks];
    if (nchunks > 0) mbar_wait(full0 + 8 * (it & 3u), (it >> 2) & 1u);
    ECHO_TRACE_MARK(p, it, 8);
    const uint32_t slot0 = (it * (uint32_t)nchunks) % C::kRing;
    // the thread's vector of the last chunk is masked once, in its own ring slot, so the unrolled copy below stays
    // branch-free (the slot is re-filled only after barrier 1 + fence.proxy.async)
    if (nchunks > 0 && (!last_valid || has_tail)) {
      const uint32_t slot = (slot0 + (uint32_t)nchunks - 1u) % C::kRing;
      const uint32_t addr = ring0 + slot * C::kChunk + my_off;
      uint4 w = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
      if (last_valid) {
        w = lds_v4(addr);
        if constexpr (C::kF32) {
          uint32_t* x = &w.x;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e >= (c1 & 3)) x[e] = 0xFF800000u;
        } else {
          w = mask_tail(w, c1 & 7);
        }
      }
      sts_v4(addr, w);
    }
#pragma unroll
    for (int c = 0; c < C::kRegChunks; ++c) {
      if (c < nchunks) {
        uint32_t slot = slot0 + (uint32_t)c;
        if (slot >= (uint32_t)C::kRing) slot -= C::kRing;
        v[c] = lds_v4(ring0 + slot * C::kChunk + my_off);
      } else {
        v[c] = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
      }
    }
    __syncwarp();
    ECHO_TRACE_MARK(p, it, 9);
    ECHO_TRACE_MARK(p, it, 10);

    ECHO_TRACE_MARK(p, it, 1);
    float mx;
    if constexpr (C::kF32) {
      float m = -INFINITY;
#pragma unroll
      for (int c = 0; c < C::kRegChunks; ++c)
        m = fmaxf(m, fmaxf(fmaxf(__uint_as_float(v[c].x), __uint_as_float(v[c].y)),
                           fmaxf(__uint_as_float(v[c].z), __uint_as_float(v[c].w))));
      mx = m;
    } else {
      uint32_t mx2 = kBf16NegInf2;
#pragma unroll
      for (int c = 0; c < C::kRegChunks; ++c) mx2 = bmax2(mx2, bmax2(bmax2(v[c].x, v[c].y), bmax2(v[c].z, v[c].w)));
      mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u));
    }
    const bool own_a = a >= col_t && a < c1 && ((a - col_t) % C::kChunkElems) < E;
    if (tid == 0 && a >= c0 && a < c1) {  // the action's logit, straight from the ring (valid until barrier 1)
      const uint32_t off = (uint32_t)(a - c0) * (uint32_t)C::kElemBytes;
      uint32_t slot = slot0 + off / C::kChunk;
      if (slot >= (uint32_t)C::kRing) slot -= C::kRing;
      const uint32_t at = ring0 + slot * C::kChunk + off % C::kChunk;
      if constexpr (C::kF32) sm.za = __uint_as_float(lds_u32(at));
      else sm.za = __uint_as_float((uint32_t)lds_u16(at) << 16);
    }

    // ---- pass 1b
    const float mb = (mx == -INFINITY) ? 0.0f : mx * kLog2e;
    const uint64_t nmb2 = f2(-mb, -mb);
    uint64_t s2 = f2(0.0f, 0.0f), t2 = f2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < C::kRegChunks; ++c) {
      if (c < nchunks) {
        uint32_t* w = &v[c].x;
#pragma unroll
        for (int k = 0; k < (C::kF32 ? 2 : 4); ++k) {  // two logits per step: a bf16 pair word, or two fp32 words
          // entropy: masked -inf logits are clamped to -1e30 so that e z = 0 (not NaN) here and in pass 2
          if constexpr (kEnt) {
            if constexpr (C::kF32) {
              w[2 * k] = __float_as_uint(fmaxf(__uint_as_float(w[2 * k]), -1.0e30f));
              w[2 * k + 1] = __float_as_uint(fmaxf(__uint_as_float(w[2 * k + 1]), -1.0e30f));
            } else {
              w[k] = bmax2(w[k], kBf16NegBig2);
            }
          }
          const uint64_t z2 = C::kF32 ? f2(__uint_as_float(w[2 * k]), __uint_as_float(w[2 * k + 1])) : bf2_to_f2(w[k]);
          float e0, e1;
          f2split(fma2(z2, l2e2, nmb2), e0, e1);
          e0 = ex2(e0);
          e1 = ex2(e1);
          s2 = add2(s2, f2(e0, e1));
          if (kEnt) t2 = fma2(f2(e0, e1), z2, t2);
          if (kStoreExp) {
            if constexpr (C::kF32) {  // fp32 logits: the exps replace them at full precision
              w[2 * k] = __float_as_uint(e0);
              w[2 * k + 1] = __float_as_uint(e1);
            } else {
              w[k] = pack_f16x2(e0, e1);
            }
          }
        }
      }
    }
    float slo, shi;
    f2split(s2, slo, shi);
    ECHO_TRACE_MARK(p, it, 11);
    float tsum = 0.0f;
    if (kEnt) {
      float tlo, thi;
      f2split(t2, tlo, thi);
      tsum = tlo + thi;
    }
    const MaxSum3 acc = kEnt ? warp_maxsum3(mx, slo + shi, tsum) : MaxSum3{warp_maxsum(MaxSum{mx, slo + shi}), 0.0f};
    if (lane == 0) {
      sm.red_m[it & 1u][warp] = acc.ms.m;
      sm.red_s[it & 1u][warp] = acc.ms.s;
      if (kEnt) sm.red_t[it & 1u][warp] = acc.t;
    }
    ECHO_TRACE_MARK(p, it, 2);
    named_bar_sync(kQBar, C::kThreads);
    ECHO_TRACE_MARK(p, it, 3);
    // every warp has copied row `it` out of the ring: warp 1 streams row it+1 into the slots (its chunks only
    // overlap rows <= it), off the critical path of warp 0's merge
    if (warp == 1) {
      if (lane == 0) {
        // every thread has read row(it) (at the top of iteration it-1): re-arm its table slot for iteration it+4
        mbar_arrive_expect_tx(rowbar0 + 8 * (it & 3u), 8);
        if (sched_thread && !sched_done) {
          const unsigned long long r = grabbed < (unsigned long long)n_rows ? grabbed : (unsigned long long)n_rows;
          broadcast(it + kRowAhead, r);
          sched_done = r >= (unsigned long long)n_rows;
          if (!sched_done) grabbed = atomicAdd(&sched[0], 1ull);
        }
      }
      if (nchunks > 0 && row_next < n_rows) {
        // iterations it+1 (row_next) and it+2; never past the first end-of-rows marker
        const int64_t r2 = row_of(it + 2);
        uint32_t upto = min((it + 1) * (uint32_t)nchunks + (uint32_t)C::kRing, (it + 3) * (uint32_t)nchunks);
        if (r2 >= n_rows) upto = min(upto, (it + 2) * (uint32_t)nchunks);
        if (upto > issued) {
          fence_proxy_async_smem();
          quad_issue_chunks<C>(p, g, issued, upto, lane, full0, ring0, policy_evict_normal(), it + 1, row_next, r2, r2);
          issued = upto;
        }
      }
    }

    // ---- CTA merge (warp 0), cluster merge (st.async to every peer), epilogue (lane 0)
    if (warp == 0) {
      const uint32_t rp = it & 1u;
      MaxSum3 mine;
      if (kEnt) {
        mine = warp_maxsum3(lane < C::kWarps ? sm.red_m[rp][lane] : -INFINITY,
                            lane < C::kWarps ? sm.red_s[rp][lane] : 0.0f, lane < C::kWarps ? sm.red_t[rp][lane] : 0.0f);
      } else {
        mine.ms = warp_maxsum(lane < C::kWarps ? MaxSum{sm.red_m[rp][lane], sm.red_s[rp][lane]}
                                               : MaxSum{-INFINITY, 0.0f});
        mine.t = 0.0f;
      }
      ECHO_TRACE_MARK(p, it, 12);
      if (lane == 0) {
        const uint32_t par = it & 1u;
        const bool owner = (a >= c0 && a < c1);
        // {m, s, t, z_a}: the receivers take z_a from the rank that owns column a (a / q)
        const uint4 msg = make_uint4(__float_as_uint(mine.ms.m), __float_as_uint(mine.ms.s), __float_as_uint(mine.t),
                                     __float_as_uint(owner ? sm.za : 0.0f));
        const uint32_t xbar_local = smem_u32(&sm.xbar[par]);
        mbar_arrive_expect_tx(xbar_local, 16 * C::kCtas);
#pragma unroll
        for (int r = 0; r < C::kCtas; ++r)
          st_async_v4(mapa(smem_u32(&sm.xbuf[par][rank]), r), msg, mapa(xbar_local, r));
        ECHO_TRACE_MARK(p, it, 6);
        finish(it, row, a);
      }
    }
    if (tid == 0) cp_async_wait<0>();  // A(it+1) landed: barrier 2 publishes row it+1's action
    named_bar_sync(kQBar, C::kThreads);
    ECHO_TRACE_MARK(p, it, 4);
    if constexpr (!kGrad) continue;
    const float coef = sm.coef, lse = sm.lse;
    const uint64_t ee2 = kEnt ? f2(sm.ent_e, sm.ent_e) : 0ull, ek2 = kEnt ? f2(sm.ent_k, sm.ent_k) : 0ull;

    // ---- pass 2
    const float kt = mx == -INFINITY ? 0.0f : -coef * ex2((mx - lse) * kLog2e);
    const uint64_t k2 = kStoreExp ? f2(kt, kt) : f2(-coef, -coef);
    const uint64_t nlse2 = f2(-lse * kLog2e, -lse * kLog2e);
    uint8_t* const row_base = p.logits + row * p.ld_bytes;
    uint8_t* const dst = row_base + (int64_t)col_t * C::kElemBytes;
    uint4 vtail = make_uint4(0u, 0u, 0u, 0u);
    const uint64_t st_pol = policy_evict_normal();
#pragma unroll
    for (int c = 0; c < C::kRegChunks; ++c) {
      if (c < nchunks) {
        uint32_t* w = &v[c].x;
#pragma unroll
        for (int k = 0; k < (C::kF32 ? 2 : 4); ++k) {
          float d0, d1;
          if (kStoreExp) {
            const uint64_t e2 = C::kF32 ? f2(__uint_as_float(w[2 * k]), __uint_as_float(w[2 * k + 1]))
                                        : f2(f16lo(w[k]), f16hi(w[k]));
            f2split(mul2(e2, k2), d0, d1);
          } else {
            const uint64_t z2 = C::kF32 ? f2(__uint_as_float(w[2 * k]), __uint_as_float(w[2 * k + 1])) : bf2_to_f2(w[k]);
            float t0, t1;
            f2split(fma2(z2, l2e2, nlse2), t0, t1);
            if (kEnt) {  // d = p (e (z - lse + H) - c) = p (e z + k),  k = e (H - lse) - c
              // (interleaved A/B, profiles/r2{j,p,t}_ab_ent.jsonl: the odd chunks' exponential on an FMA-pipe
              // polynomial was 17 % slower; a tile with twice the threads per row caching both z and e, 21 % slower;
              // the exps written back over the logits in the ring slots and read in pass 2, 19 % slower)
              f2split(mul2(f2(ex2(t0), ex2(t1)), fma2(z2, ee2, ek2)), d0, d1);
            }
            else
              f2split(mul2(f2(ex2(t0), ex2(t1)), k2), d0, d1);
          }
          if constexpr (C::kF32) {
            w[2 * k] = __float_as_uint(d0);
            w[2 * k + 1] = __float_as_uint(d1);
          } else {
            w[k] = pack_bf16x2(d0, d1);
          }
        }
        if (c < nstore) stg_v4_hint(dst + (int64_t)c * C::kChunk, v[c], st_pol);
        if (c == nchunks - 1) vtail = v[c];
      }
    }
    // one partial store after the unrolled loop (not one copy per chunk): keeps the loop body in the I-cache
    if (has_tail) {
      uint8_t* const tail = dst + (int64_t)(nchunks - 1) * C::kChunk;
      if constexpr (C::kF32) {
        const uint32_t tw[4] = {vtail.x, vtail.y, vtail.z, vtail.w};
#pragma unroll
        for (int e = 0; e < 3; ++e)
          if (e < (c1 & 3)) reinterpret_cast<uint32_t*>(tail)[e] = tw[e];
      } else {
        store_partial8(reinterpret_cast<__nv_bfloat16*>(tail), vtail, c1 & 7);
      }
    }
    ECHO_TRACE_MARK(p, it, 5);
    if (own_a) {
      if constexpr (C::kF32) reinterpret_cast<float*>(row_base)[a] = sm.da;
      else reinterpret_cast<__nv_bfloat16*>(row_base)[a] = __float2bfloat16_rn(sm.da);
    }
  }
  cluster_sync_all();
  if (tid == 0) {
    // the last CTA out resets this launch's scheduler slot (all grabs returned before the cluster barrier)
    __threadfence();
    if (atomicAdd(&sched[1], 1ull) == (unsigned long long)gridDim.x - 1ull) {
      sched[0] = 0ull;
      sched[1] = 0ull;
    }
  }
}

template <class C>
static bool supports_t(int32_t dtype, int32_t V) {
  constexpr int32_t E = C::kVecElems;
  if (dtype != (C::kF32 ? ECHO_F32 : ECHO_BF16) || V < E * C::kCtas) return false;
  const int32_t q = ((V + C::kCtas - 1) / C::kCtas + E - 1) & ~(E - 1);
  return ((int64_t)q * C::kElemBytes + C::kChunk - 1) / C::kChunk <= C::kRegChunks;
}

template <class C, int kMode>
static cudaError_t launch_t(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  const size_t smem = sizeof(QuadSmem<C>);
  const void* fn = (const void*)policy_loss_quad_kernel<C, kMode>;
  // function attributes and the resident-cluster count are per device and never change: set / query once
  static std::atomic<int> cached[kMaxDevices];  // resident clusters + 1 (0: not yet known)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int64_t clusters = dev < kMaxDevices ? (int64_t)cached[dev].load(std::memory_order_relaxed) - 1 : -1;
  if (clusters < 0) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (C::kCtas > 8) {  // 16-CTA clusters are beyond the portable size: opt in
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    clusters = max_active_clusters(fn, C::kThreads, smem, C::kCtas, num_sms * C::kCtasPerSm / C::kCtas);
    if (dev < kMaxDevices) cached[dev].store((int)clusters + 1, std::memory_order_relaxed);
  }
  if (clusters > p.n_rows) clusters = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)(clusters * C::kCtas), C::kCtas, C::kThreads, (int32_t)smem};
    return cudaSuccess;
  }
  LossParams q = p;
  q.sched_slot = (int32_t)next_sched_slot(g_next_sched_slot, g_next_sched_slot_graph, stream, kSchedSlots);
  policy_loss_quad_kernel<C, kMode><<<(unsigned)(clusters * C::kCtas), C::kThreads, smem, stream>>>(q);
  return cudaGetLastError();
}

using Quad = QCfg<4, 8>;
using Oct = QCfg<8, 4>;
using Hex = QCfg<16, 4>;  // 16-CTA cluster (non-portable size): vocabularies up to 311296 (Gemma / Llama-4 class)
using HexF = QCfg<16, 4, true>;  // 16-CTA cluster over fp32 logits: vocabularies up to 155648

bool quad_supports(int32_t dtype, int32_t V) { return supports_t<Quad>(dtype, V); }
bool oct_supports(int32_t dtype, int32_t V) { return supports_t<Oct>(dtype, V); }
bool hex_supports(int32_t dtype, int32_t V) {
  return dtype == ECHO_F32 ? supports_t<HexF>(dtype, V) : supports_t<Hex>(dtype, V);
}

static bool wants_entropy(const LossParams& p) { return p.entropy_coef > 0.0f || p.tok_entropy != nullptr; }
cudaError_t launch_quad(const LossParams& p, bool store_exp, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  if (wants_entropy(p)) return launch_t<Quad, kModeEntropy>(p, stream, num_sms, shape);
  return store_exp ? launch_t<Quad, kModeCache>(p, stream, num_sms, shape)
                   : launch_t<Quad, kModeExact>(p, stream, num_sms, shape);
}
cudaError_t launch_oct(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  if (wants_entropy(p)) return launch_t<Oct, kModeEntropy>(p, stream, num_sms, shape);
  return launch_t<Oct, kModeCache>(p, stream, num_sms, shape);
}
cudaError_t launch_hex(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  if (dtype == ECHO_F32) {
    if (wants_entropy(p)) return launch_t<HexF, kModeEntropy>(p, stream, num_sms, shape);
    return launch_t<HexF, kModeCache>(p, stream, num_sms, shape);
  }
  if (wants_entropy(p)) return launch_t<Hex, kModeEntropy>(p, stream, num_sms, shape);
  return launch_t<Hex, kModeCache>(p, stream, num_sms, shape);
}
// forward-only log-probs: the 8-CTA tile (1.93 ms vs 1.97 ms for the 4-CTA one on 32768 x 151936), the 16-CTA
// tile past its vocabulary range
#ifdef ECHO_LOGP_HEX8
using HexLogp = QCfg<16, 4, false, 10, 8>;
#endif
cudaError_t launch_quad_logp(const LossParams& p, int32_t dtype, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  if (dtype == ECHO_F32) return launch_t<HexF, kModeLogp>(p, stream, num_sms, shape);
#ifdef ECHO_LOGP_HEX8
  if (supports_t<HexLogp>(ECHO_BF16, p.V)) return launch_t<HexLogp, kModeLogp>(p, stream, num_sms, shape);
#endif
  if (!supports_t<Oct>(ECHO_BF16, p.V)) return launch_t<Hex, kModeLogp>(p, stream, num_sms, shape);
  return launch_t<Oct, kModeLogp>(p, stream, num_sms, shape);
}

}  // namespace echo
