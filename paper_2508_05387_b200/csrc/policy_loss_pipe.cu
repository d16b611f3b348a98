// policy_loss_pipe.cu -- ECHO_ALGO_PIPE: the B200 design of the fused (3)+(4)+(5) kernel.
//
// One CTA per SM owns whole rows (persistent, rows strided by CTA) and runs a three-role warp-specialised
// pipeline, so that the row-level dependency (the gradient of every logit needs the log-sum-exp of the whole
// row) never serialises the SM:
//
//   producer (1 warp, one lane)  1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx) feed two
//                                shared-memory rings: ring R streams row k+1 from HBM (L2 evict_last, so the
//                                row stays in L2), ring W streams row k a second time from L2 (evict_first)
//   reducers (7 warps)           pass 1 on row k+1 out of ring R: exact bf16x2 chunk max, online rescaled
//                                sum of 2^((z - m) log2e) (MUFU) in fp32, warp shuffles -> CTA merge in a
//                                fixed order -> lse, logp, rho, clip, KL, c_t -> a double-buffered mailbox
//   writers (8 warps)            pass 2 on row k out of ring W: d = -c_t 2^((z - lse) log2e) (MUFU), bf16 RNE,
//                                16-byte stores in place; the action column gets c_t (1 - p_a)
//
// HBM traffic is one read (ring R) and one write per logit; the second read is an L2 hit because a row is
// re-read ~one row-time after it was first streamed (~45 MB of rows in flight chip-wide, well inside the
// 126 MB L2).  No clusters, no DSMEM: every row is reduced inside one SM, in an order fixed by V alone.
#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"
#include "policy_loss_common.cuh"

namespace echo {

constexpr int kPRedWarps = 7;
constexpr int kPWrtWarps = 8;
constexpr int kPRed = kPRedWarps * 32;                  // 224 reducer threads
constexpr int kPWrt = kPWrtWarps * 32;                  // 256 writer threads
constexpr int kPThreads = kPRed + kPWrt + 32;           // + producer warp = 512 (4 warps per SMSP)
constexpr int kPChunkR = kPRed * 32;                    // 7168 B: two 16-byte vectors per reducer thread
constexpr int kPChunkW = kPWrt * 32;                    // 8192 B: two 16-byte vectors per writer thread
constexpr int kPRingR = 16;                             // 112 KB
constexpr int kPRingW = 12;                             // 96 KB
constexpr int kPBarRed = 1;                             // named barrier of the reducer warps

struct Mail {
  float lse_l2e, coef, da, pad;
};

struct __align__(128) PipeSmem {
  uint8_t ring_r[kPRingR][kPChunkR];
  uint8_t ring_w[kPRingW][kPChunkW];
  uint64_t full_r[kPRingR], empty_r[kPRingR];
  uint64_t full_w[kPRingW], empty_w[kPRingW];
  uint64_t mail_full[2], mail_empty[2];
  Mail mail[2];
  float red_m[kPRedWarps], red_s[kPRedWarps];
  float za[2];
};

// Online (max, sum-exp) update with one 16-byte vector of 8 bf16 logits; lanes are fp32 pairs.
ECHO_DEVINL void online8(float& m, uint64_t& s2, const uint4& w, uint64_t l2e2) {
  const uint32_t c2 = bmax2(bmax2(w.x, w.y), bmax2(w.z, w.w));
  const float cm = fmaxf(__uint_as_float(c2 << 16), __uint_as_float(c2 & 0xFFFF0000u));
  if (cm > m) {  // rare after the first few vectors of a row
    const float f = (m == -INFINITY) ? 0.0f : ex2((m - cm) * kLog2e);
    s2 = mul2(s2, f2(f, f));
    m = cm;
  }
  const float mb = (m == -INFINITY) ? 0.0f : m * kLog2e;
  const uint64_t nmb2 = f2(-mb, -mb);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float e0, e1;
    f2split(fma2(bf2_to_f2(ws[k]), l2e2, nmb2), e0, e1);
    s2 = add2(s2, f2(ex2(e0), ex2(e1)));
  }
}

__global__ void __launch_bounds__(kPThreads, 1) policy_loss_pipe_kernel(const LossParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PipeSmem& sm = *reinterpret_cast<PipeSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t V = p.V;
  const uint32_t row_bytes = (uint32_t)((V + 7) & ~7) * 2u;  // bytes loaded per row (16-byte multiple)
  const int nch_r = (int)((row_bytes + kPChunkR - 1) / kPChunkR);
  const int nch_w = (int)((row_bytes + kPChunkW - 1) / kPChunkW);
  const uint32_t my_rows =
      p.n_rows > (int64_t)blockIdx.x ? (uint32_t)((p.n_rows - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
  const uint32_t fr0 = smem_u32(&sm.full_r[0]), er0 = smem_u32(&sm.empty_r[0]);
  const uint32_t fw0 = smem_u32(&sm.full_w[0]), ew0 = smem_u32(&sm.empty_w[0]);
  const uint32_t rr0 = smem_u32(&sm.ring_r[0][0]), rw0 = smem_u32(&sm.ring_w[0][0]);
  const uint32_t mf0 = smem_u32(&sm.mail_full[0]), me0 = smem_u32(&sm.mail_empty[0]);

  if (tid == 0) {
    for (int i = 0; i < kPRingR; ++i) {
      mbar_init(fr0 + 8 * i, 1);
      mbar_init(er0 + 8 * i, kPRedWarps);
    }
    for (int i = 0; i < kPRingW; ++i) {
      mbar_init(fw0 + 8 * i, 1);
      mbar_init(ew0 + 8 * i, kPWrtWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(mf0 + 8 * i, 1);
      mbar_init(me0 + 8 * i, kPWrtWarps);
    }
    fence_mbar_init_cluster();
  }
  __syncthreads();

  if (warp == kPRedWarps + kPWrtWarps) {
    // ============================================================ producer
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
      const uint32_t tot_r = my_rows * (uint32_t)nch_r, tot_w = my_rows * (uint32_t)nch_w;
      uint32_t sr = 0, sw = 0;  // next chunk of each stream
      while (sr < tot_r || sw < tot_w) {
        if (sr < tot_r) {
          const uint32_t slot = sr % kPRingR, ph = (sr / kPRingR) & 1u;
          if (mbar_try_wait(er0 + 8 * slot, ph ^ 1u)) {
            const uint32_t r = sr / (uint32_t)nch_r, c = sr % (uint32_t)nch_r;
            const int64_t row = (int64_t)blockIdx.x + (int64_t)r * gridDim.x;
            const uint32_t nb = min((uint32_t)kPChunkR, row_bytes - c * kPChunkR);
            mbar_arrive_expect_tx(fr0 + 8 * slot, nb);
            bulk_g2s(rr0 + slot * kPChunkR, p.logits + row * p.ld_bytes + (int64_t)c * kPChunkR, nb, fr0 + 8 * slot,
                     pol_keep);
            ++sr;
          }
        }
        // the second read of row r starts only after its first read has been issued in full (L2 hit)
        if (sw < tot_w && (sw / (uint32_t)nch_w + 1) * (uint32_t)nch_r <= sr) {
          const uint32_t slot = sw % kPRingW, ph = (sw / kPRingW) & 1u;
          if (mbar_try_wait(ew0 + 8 * slot, ph ^ 1u)) {
            const uint32_t r = sw / (uint32_t)nch_w, c = sw % (uint32_t)nch_w;
            const int64_t row = (int64_t)blockIdx.x + (int64_t)r * gridDim.x;
            const uint32_t nb = min((uint32_t)kPChunkW, row_bytes - c * kPChunkW);
            mbar_arrive_expect_tx(fw0 + 8 * slot, nb);
            bulk_g2s(rw0 + slot * kPChunkW, p.logits + row * p.ld_bytes + (int64_t)c * kPChunkW, nb, fw0 + 8 * slot,
                     pol_drop);
            ++sw;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kPRedWarps) {
    // ============================================================ reducers: pass 1 + epilogue
    const int t = tid;
    const float gscale = (float)((double)p.grad_scale / *p.n_global);
    const uint64_t l2e2 = f2(kLog2e, kLog2e);
    uint32_t seq = 0;
    for (uint32_t it = 0; it < my_rows; ++it) {
      const int64_t row = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const int32_t a = p.tok_action[row];
      RowMeta meta{0.f, 0.f, 0.f};
      if (t == 0) meta = load_meta(p, row);
      const uint32_t par = it & 1u;
      float m = -INFINITY;
      uint64_t s2 = f2(0.0f, 0.0f);
      for (int c = 0; c < nch_r; ++c, ++seq) {
        const uint32_t slot = seq % kPRingR, ph = (seq / kPRingR) & 1u;
        mbar_wait(fr0 + 8 * slot, ph);
        uint4 w[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) w[h] = lds_v4(rr0 + slot * kPChunkR + h * (kPChunkR / 2) + t * 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(er0 + 8 * slot);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t boff = (uint32_t)c * kPChunkR + h * (kPChunkR / 2) + t * 16;  // byte offset in the row
          const int32_t col = (int32_t)(boff >> 1);
          if (boff >= row_bytes) continue;
          if (col + 8 > V) w[h] = mask_tail(w[h], V - col);
          if ((uint32_t)(a - col) < 8u) {
            const int e = a - col;
            const uint32_t word = e < 2 ? w[h].x : e < 4 ? w[h].y : e < 6 ? w[h].z : w[h].w;
            sm.za[par] = (e & 1) ? __uint_as_float(word & 0xFFFF0000u) : __uint_as_float(word << 16);
          }
          online8(m, s2, w[h], l2e2);
        }
      }
      float slo, shi;
      f2split(s2, slo, shi);
      const MaxSum acc = warp_maxsum(MaxSum{m, slo + shi});
      if (lane == 0) {
        sm.red_m[warp] = acc.m;
        sm.red_s[warp] = acc.s;
      }
      named_bar_sync(kPBarRed, kPRed);
      if (warp == 0) {
        MaxSum tot = lane < kPRedWarps ? MaxSum{sm.red_m[lane], sm.red_s[lane]} : MaxSum{-INFINITY, 0.0f};
        tot = warp_maxsum(tot);
        if (lane == 0) {
          const float lse = tot.m + logf(tot.s);
          const float za = (a < 0 || a >= V) ? NAN : sm.za[par];
          const RowScalars r = row_epilogue_f(lse, za, meta.old, meta.ref, meta.adv, p.clip_low, p.clip_high,
                                              p.kl_coef, gscale);
          p.tok_logp[row] = r.logp;
          p.tok_loss[row] = r.loss;
          p.tok_flags[row] = r.flags;
          const float pa = ex2(fmaf(za, kLog2e, -lse * kLog2e));
          mbar_wait(me0 + 8 * par, ((it >> 1) & 1u) ^ 1u);  // writers are done with row it - 2
          sm.mail[par] = Mail{lse * kLog2e, r.coef, fmaf(-r.coef, pa, r.coef), 0.0f};
          mbar_arrive(mf0 + 8 * par);
        }
      }
      named_bar_sync(kPBarRed, kPRed);  // red_m / red_s / za reuse
    }
  } else {
    // ============================================================ writers: pass 2
    const int t = tid - kPRed;
    const int wwarp = warp - kPRedWarps;
    const uint64_t st_pol = policy_evict_first();
    const uint64_t l2e2 = f2(kLog2e, kLog2e);
    uint32_t seq = 0;
    for (uint32_t it = 0; it < my_rows; ++it) {
      const int64_t row = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const int32_t a = p.tok_action[row];
      const uint32_t par = it & 1u;
      mbar_wait(mf0 + 8 * par, (it >> 1) & 1u);
      const Mail mail = sm.mail[par];
      __syncwarp();
      if (lane == 0) mbar_arrive(me0 + 8 * par);
      const uint64_t nlse2 = f2(-mail.lse_l2e, -mail.lse_l2e);
      const uint64_t k2 = f2(-mail.coef, -mail.coef);
      uint8_t* const row_base = p.logits + row * p.ld_bytes;
      for (int c = 0; c < nch_w; ++c, ++seq) {
        const uint32_t slot = seq % kPRingW, ph = (seq / kPRingW) & 1u;
        mbar_wait(fw0 + 8 * slot, ph);
        uint4 w[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) w[h] = lds_v4(rw0 + slot * kPChunkW + h * (kPChunkW / 2) + t * 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(ew0 + 8 * slot);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t boff = (uint32_t)c * kPChunkW + h * (kPChunkW / 2) + t * 16;
          const int32_t col = (int32_t)(boff >> 1);
          if (boff >= row_bytes) continue;
          uint32_t ws[4] = {w[h].x, w[h].y, w[h].z, w[h].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float t0, t1, d0, d1;
            f2split(fma2(bf2_to_f2(ws[k]), l2e2, nlse2), t0, t1);
            f2split(mul2(f2(ex2(t0), ex2(t1)), k2), d0, d1);
            ws[k] = pack_bf16x2(d0, d1);
          }
          const uint4 o = make_uint4(ws[0], ws[1], ws[2], ws[3]);
          if (col + 8 <= V)
            stg_v4_hint(row_base + boff, o, st_pol);
          else
            store_partial8(reinterpret_cast<__nv_bfloat16*>(row_base + boff), o, V - col);
          if ((uint32_t)(a - col) < 8u)  // same thread, same address, program order: overwrite the action column
            reinterpret_cast<__nv_bfloat16*>(row_base)[a] = __float2bfloat16_rn(mail.da);
        }
      }
      (void)wwarp;
    }
  }
}

cudaError_t launch_pipe(const LossParams& p, cudaStream_t stream, int num_sms, LaunchShape* shape) {
  const size_t smem = sizeof(PipeSmem);
  cudaError_t e = cudaFuncSetAttribute(policy_loss_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = num_sms;
  if (grid > p.n_rows) grid = p.n_rows;
  if (shape) {
    *shape = LaunchShape{(int32_t)grid, 1, kPThreads, (int32_t)smem};
    return cudaSuccess;
  }
  policy_loss_pipe_kernel<<<(unsigned)grid, kPThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace echo
