// token_logp.cu -- f1: forward-only log-probs logp_t = z[t, a_t] - logsumexp_v z[t, v] over bf16
// logits, read once (PAPER.md :170 -- the log pi(a|s) each rollout carries; :278 the reference model of KL-PPO).
//
// One WARP per row, no CTA or cluster barrier.  Read-only, the row never has to be held for a second pass, so there
// is nothing to gain from splitting it over a cluster (the fused (3)-(5) kernel does that to keep the row in
// registers between its read and its write): each of the 16 warps of a CTA streams its own row through a private
// 2 x 6 KB shared-memory ring filled by 1-D TMA bulk copies (lane 0 issues them kStages chunks ahead, across row
// boundaries), and keeps an online max / sum of 2^((z - m) log2e) per lane -- one MUFU per logit, a rescale only when
// a lane's running max grows.  At the row's end a fixed shuffle tree merges the 32 lanes (deterministic: the order
// depends only on V), and lane 0 writes logp, lse and the non-finite flag.  Rows are taken in order from a global
// counter, so the warps of the whole GPU stream one compact window of rows.
#include <cuda_bf16.h>

#include <stdlib.h>

#include <atomic>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

namespace tl {
constexpr int kWarps = 16, kThreads = kWarps * 32;
template <int kStages, int kChunk>  // 2 x 6 KB (3072 bf16 logits) per warp by default: 192 KB per SM
struct alignas(128) WarpRing {
  uint8_t buf[kStages][kChunk];
  uint64_t full[kStages];
  int64_t row[kStages];    // the (row, chunk) each slot holds (row < 0: no more work)
  int32_t chunk[kStages];
};
template <int kStages, int kChunk>
struct Smem {
  WarpRing<kStages, kChunk> ring[kWarps];
};
constexpr int kSlots = 256;
}  // namespace tl

__device__ unsigned long long g_logp_sched[tl::kSlots][2];  // {next row, warps done} per launch slot
static std::atomic<uint32_t> g_logp_slot{0}, g_logp_slot_graph{0};

template <int kStages, int kChunk>
__global__ void __launch_bounds__(tl::kThreads, 1) token_logp_warp_kernel(const LossParams p) {
  using namespace tl;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<kStages, kChunk>& sm = *reinterpret_cast<Smem<kStages, kChunk>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpRing<kStages, kChunk>& rg = sm.ring[warp];
  unsigned long long* const sched = g_logp_sched[p.sched_slot];
  const int32_t V = p.V;
  const uint32_t row_bytes = (uint32_t)V * 2u;
  const uint32_t load_bytes = (row_bytes + 15u) & ~15u;             // ld * 2 >= this (16-byte multiple)
  const int32_t n_chunks = (int32_t)((load_bytes + kChunk - 1) / kChunk);
  const int64_t n_rows = p.n_rows;
  const uint32_t full0 = smem_u32(&rg.full[0]);
  const uint64_t pol = policy_evict_first();                         // read once: keep L2 for the neighbours

  // producer state (lane 0): the next (row, chunk) to issue
  int64_t prow = -1;
  int32_t pchunk = n_chunks;
  auto produce = [&](int s) {  // fill slot s with the next item (or mark the end)
    if (pchunk == n_chunks) {
      const unsigned long long r = atomicAdd(&sched[0], 1ull);
      prow = r < (unsigned long long)n_rows ? (int64_t)r : -1;
      pchunk = 0;
    }
    rg.row[s] = prow;
    rg.chunk[s] = pchunk;
    if (prow >= 0) {
      const uint32_t off = (uint32_t)pchunk * kChunk;
      const uint32_t nb = min((uint32_t)kChunk, load_bytes - off);
      mbar_arrive_expect_tx(full0 + 8 * s, nb);
      bulk_g2s(smem_u32(rg.buf[s]), p.logits + prow * p.ld_bytes + off, nb, full0 + 8 * s, pol);
      ++pchunk;
    } else {
      mbar_arrive(full0 + 8 * s);  // completes the phase: the consumer sees row < 0 and stops
    }
  };
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(full0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kStages; ++s) produce(s);
  }
  __syncwarp();

  const uint64_t l2e2 = f2(kLog2e, kLog2e);
  float m = -INFINITY, ssum = 0.0f;  // this lane's running max and sum of 2^((z - m) log2e)
  float za = 0.0f;
  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % kStages);
    mbar_wait(full0 + 8 * s, (it / kStages) & 1u);
    const int64_t row = rg.row[s];
    if (row < 0) break;
    const int32_t chunk = rg.chunk[s];
    if (chunk == 0) {
      m = -INFINITY;
      ssum = 0.0f;
      if (lane == 0) {
        const int32_t a = p.tok_action[row];
        za = (a >= 0 && a < V) ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.logits + row * p.ld_bytes)[a])
                               : NAN;
      }
    }
    // this lane's vectors of the chunk: l, l + 32, ... (8 bf16 each; conflict-free LDS.128).  The chunk's exps go
    // to a packed pair of chunk-local accumulators that joins the running sum once per chunk: the sequential fp32
    // chain stays ~(V / 2048 + 32) adds long instead of V / 256, which keeps logp within ~1e-6 of fp64 at V = 311296
    const int32_t col0 = chunk * (kChunk / 2);
    uint64_t acc = f2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < kChunk / 16 / 32; ++k) {
      const int32_t col = col0 + (k * 32 + lane) * 8;
      if (col >= V) break;
      uint4 w = lds_v4(smem_u32(rg.buf[s]) + (uint32_t)(k * 32 + lane) * 16u);
      if (col + 8 > V) w = mask_tail(w, V - col);
      const uint32_t mx2 = bmax2(bmax2(w.x, w.y), bmax2(w.z, w.w));
      const float mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xFFFF0000u));
      if (mx > m) {  // the running max grows (rare after the first vectors): rescale both sums
        const float f = (m == -INFINITY) ? 0.0f : ex2((m - mx) * kLog2e);
        ssum *= f;
        acc = mul2(acc, f2(f, f));
        m = mx;
      }
      const float mb = (m == -INFINITY) ? 0.0f : m * kLog2e;
      const uint64_t nmb2 = f2(-mb, -mb);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float e0, e1;
        f2split(fma2(bf2_to_f2(ws[j]), l2e2, nmb2), e0, e1);
        acc = add2(acc, f2(ex2(e0), ex2(e1)));
      }
    }
    {
      float lo, hi;
      f2split(acc, lo, hi);
      ssum += lo + hi;
    }
    __syncwarp();  // every lane is done with slot s
    if (lane == 0) {
      fence_proxy_async_smem();  // the generic-proxy reads of slot s before the TMA write that refills it
      produce(s);
    }
    if (chunk == n_chunks - 1) {
      // the row's lse: max over lanes first, then the rescaled sums, fixed xor tree (deterministic)
      float M = m;
#pragma unroll
      for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
      float S = (m == -INFINITY) ? 0.0f : ssum * ex2((m - M) * kLog2e);
#pragma unroll
      for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xFFFFFFFFu, S, o);
      if (lane == 0) {
        const float lse = M + logf(S);
        const float logp = za - lse;
        p.tok_logp[row] = logp;
        if (p.tok_lse) p.tok_lse[row] = lse;
        if (p.tok_flags) p.tok_flags[row] = (isfinite(lse) && isfinite(logp)) ? 0 : ECHO_FLAG_NONFINITE;
      }
    }
  }
  // the last warp out resets this launch's scheduler slot
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(&sched[1], 1ull) == (unsigned long long)gridDim.x * kWarps - 1ull) {
      sched[0] = 0ull;
      sched[1] = 0ull;
      __threadfence();
    }
  }
}

bool token_logp_warp_supports(int32_t dtype, int32_t V) { return dtype == ECHO_BF16 && V >= 8192; }

template <int kStages, int kChunk>
static cudaError_t launch_ring(const LossParams& p, cudaStream_t stream, int num_sms) {
  const size_t smem = sizeof(tl::Smem<kStages, kChunk>);
  static std::atomic<int> attr_set{0};
  if (!attr_set.load(std::memory_order_relaxed)) {
    const cudaError_t e = cudaFuncSetAttribute(token_logp_warp_kernel<kStages, kChunk>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.store(1, std::memory_order_relaxed);
  }
  LossParams q = p;
  q.sched_slot = (int32_t)next_sched_slot(g_logp_slot, g_logp_slot_graph, stream, tl::kSlots);
  int64_t grid = num_sms;
  const int64_t need = (p.n_rows + tl::kWarps - 1) / tl::kWarps;
  if (grid > need) grid = need;
  token_logp_warp_kernel<kStages, kChunk><<<(unsigned)grid, tl::kThreads, smem, stream>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_token_logp_warp(const LossParams& p, cudaStream_t stream, int num_sms) {
  // per-warp ring of 12 KB (192 KB per SM): 2 x 6 KB by default.  Interleaved A/B on one 32768 x 151936 micro-batch
  // (profiles/r2q_ab_logp.jsonl): 2 x 6 KB 1.544 ms, 3 x 4 KB 1.633, 4 x 3 KB 1.711, 6 x 2 KB 1.897 -- fewer, longer
  // bulk copies per byte; ECHO_LOGP_RING=3 / 4 / 6 selects the others
  const char* env = getenv("ECHO_LOGP_RING");
  const int ring = env ? atoi(env) : 2;
  if (ring == 3) return launch_ring<3, 4096>(p, stream, num_sms);
  if (ring == 4) return launch_ring<4, 3072>(p, stream, num_sms);
  if (ring == 6) return launch_ring<6, 2048>(p, stream, num_sms);
  return launch_ring<2, 6144>(p, stream, num_sms);
}

}  // namespace echo
