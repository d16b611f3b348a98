// echo_common.cuh -- sm_100a device helpers shared by the libecho kernels (inline PTX).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "echo.h"

#define ECHO_DEVINL __device__ __forceinline__

namespace echo {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- bf16 <-> fp32 (bit level)
ECHO_DEVINL float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
ECHO_DEVINL float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
// Two fp32 -> packed bf16x2, round-to-nearest-even (F2FP.BF16.F32.PACK_AB).  `lo` lands in bits 0..15.
ECHO_DEVINL uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Two fp32 -> packed f16x2 (RNE); `lo` lands in bits 0..15.  And back.
ECHO_DEVINL uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
ECHO_DEVINL float f16lo(uint32_t w) {
  float f;
  asm("{\n\t.reg .f16 h;\n\tmov.b32 {h, _}, %1;\n\tcvt.f32.f16 %0, h;\n\t}" : "=f"(f) : "r"(w));
  return f;
}
ECHO_DEVINL float f16hi(uint32_t w) {
  float f;
  asm("{\n\t.reg .f16 h;\n\tmov.b32 {_, h}, %1;\n\tcvt.f32.f16 %0, h;\n\t}" : "=f"(f) : "r"(w));
  return f;
}

// ---------------------------------------------------------------- packed helpers (Blackwell f32x2 pipes)
// A pair of fp32 lives in one 64-bit register pair; fma/add/mul.rn.f32x2 issue as one FFMA2/FADD2/FMUL2.
ECHO_DEVINL uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
ECHO_DEVINL void f2split(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
ECHO_DEVINL uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
ECHO_DEVINL uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
ECHO_DEVINL uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// bf16x2 word -> fp32 pair (exact)
ECHO_DEVINL uint64_t bf2_to_f2(uint32_t w) { return f2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u)); }
// max of two bf16x2 words (exact; a NaN operand yields the other operand)
ECHO_DEVINL uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
constexpr uint32_t kBf16NegInf2 = 0xFF80FF80u;
constexpr uint32_t kBf16NegBig2 = 0xF14AF14Au;  // bf16 -1.0e30 twice: the entropy path's stand-in for -inf

ECHO_DEVINL float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------- L2 cache policies
ECHO_DEVINL uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
ECHO_DEVINL uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
ECHO_DEVINL uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

ECHO_DEVINL uint4 ldg_v4_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
ECHO_DEVINL void stg_v4_hint(void* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------- shared-memory addressing
ECHO_DEVINL uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

ECHO_DEVINL uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
ECHO_DEVINL uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
ECHO_DEVINL uint16_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
ECHO_DEVINL void sts_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// 4-byte global -> shared copies without a register round trip (LDGSTS), in commit groups
ECHO_DEVINL void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
ECHO_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
ECHO_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- mbarrier
ECHO_DEVINL void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
ECHO_DEVINL void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
ECHO_DEVINL void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
ECHO_DEVINL void mbar_arrive_expect_tx(uint32_t bar, uint32_t tx) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
               "r"(tx)
               : "memory");
}
ECHO_DEVINL bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
ECHO_DEVINL void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Acquire at cluster scope: for data written into this CTA's smem by the peer CTA (st.async).
ECHO_DEVINL bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
ECHO_DEVINL void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
// A whole warp waits on one barrier: lane 0 polls it, then every lane takes its own (now immediate) acquire.
// (try_wait suspend-time hints on the tensor-core kernels' waits were neutral to 25 % slower in interleaved A/B:
// profiles/r2j_ab_cublas.jsonl, r2l_ab_cublas.jsonl.)
ECHO_DEVINL void mbar_wait_cluster_warp(uint32_t bar, uint32_t parity, int lane) {
  if (lane == 0) mbar_wait_cluster(bar, parity);
  __syncwarp();
  mbar_wait_cluster(bar, parity);
}

// ---------------------------------------------------------------- bulk async copy (TMA, 1-D)
// global -> this CTA's shared memory, completion signalled on `bar` (complete_tx::bytes).
ECHO_DEVINL void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

// Order this thread's earlier generic-proxy shared-memory accesses (and, after a CTA barrier, those of the
// threads it synchronised with) before its subsequent async-proxy (TMA) accesses.
ECHO_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------- clusters / DSMEM
ECHO_DEVINL uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
ECHO_DEVINL uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
ECHO_DEVINL uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
ECHO_DEVINL uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
ECHO_DEVINL void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16-byte remote store into the peer CTA's smem that completes 16 tx-bytes on the peer's mbarrier.
ECHO_DEVINL void st_async_v4(uint32_t remote_addr, uint4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                   remote_addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(remote_bar)
               : "memory");
}

ECHO_DEVINL void st_async_b64(uint32_t remote_addr, uint64_t v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr), "l"(v),
               "r"(remote_bar)
               : "memory");
}

// ---------------------------------------------------------------- named barriers
ECHO_DEVINL void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- online (max, sum-exp) pair
// Merge is symmetric bit-for-bit (IEEE add/mul commute), so butterfly reductions give every lane the
// same value; the order of a tree depends only on thread layout.
struct MaxSum {
  float m;  // running max (-inf when empty)
  float s;  // sum of exp(x - m)
};
ECHO_DEVINL MaxSum maxsum_merge(MaxSum a, MaxSum b) {
  float m = fmaxf(a.m, b.m);
  if (m == -INFINITY) return MaxSum{m, a.s + b.s};
  float sa = a.s * ex2((a.m - m) * kLog2e);
  float sb = b.s * ex2((b.m - m) * kLog2e);
  return MaxSum{m, sa + sb};
}
// Warp merge with ONE exponential per lane on the critical path: butterfly max, rescale, butterfly sum.
// (A pairwise-merge butterfly would chain 5 dependent MUFU ops, each queued behind the bulk pass-1b exps of
// the other warps on the SM.)  IEEE add/max commute, so every lane ends with the same bits.
ECHO_DEVINL MaxSum warp_maxsum(MaxSum v) {
  float mx = v.m;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float t = (v.m == -INFINITY) ? 0.0f : v.s * ex2((v.m - mx) * kLog2e);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return MaxSum{mx, t};
}

// (m, s, t) with t = sum x e^{x - m}: the entropy path's third accumulator, rescaled like s.
struct MaxSum3 {
  MaxSum ms;
  float t;
};
ECHO_DEVINL MaxSum3 warp_maxsum3(float m, float s, float t) {
  float mx = m;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float f = (m == -INFINITY) ? 0.0f : ex2((m - mx) * kLog2e);
  float ss = s * f, tt = t * f;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    tt += __shfl_xor_sync(0xffffffffu, tt, o);
  }
  return MaxSum3{MaxSum{mx, ss}, tt};
}

// ---------------------------------------------------------------- the per-row scalar epilogue (4)
struct RowScalars {
  float logp, loss, coef;  // coef = c_t: dl/dlogp * scale  (scale = grad_scale * w_t, w_t = 1/N_global or tok_weight)
  float ecoef;             // scale * eta: the entropy term's gradient factor (0 when off)
  uint8_t flags;
};
struct LossOpts {
  float clip_low, clip_high, clip_dual, kl_coef;
  int32_t kl_estimator;  // ECHO_KL_K3 | ECHO_KL_K1 | ECHO_KL_K2
  float entropy_coef;    // eta (0 = off)
};
// lse: log-sum-exp of the row; za: logit at the action; adv: the token's advantage; scale: grad_scale * w_t.
//   rho = exp(logp - old); pg = max(-A rho, -A clip(rho, 1-lo, 1+hi)) (SPEC.md :219); dual clip (A < 0,
//   rho > c): pg = -A c; KL to pi_ref by the selected estimator (x = ref - logp): k3 e^x - x - 1 (default),
//   k1 -x, k2 x^2/2; l_t = pg + beta kl - eta H (H: the row's entropy, only read when eta > 0);
//   c_t = scale * ([not clipped](-A rho) + beta dkl/dlogp).
ECHO_DEVINL RowScalars row_epilogue(float lse, float za, float old, float ref, float adv, const LossOpts& o,
                                    float scale, float H = 0.0f) {
  RowScalars r;
  const float logp = za - lse;
  const float rho = expf(logp - old);
  const float lo = 1.0f - o.clip_low, hi = 1.0f + o.clip_high;
  bool clipped = (adv > 0.0f && rho > hi) || (adv < 0.0f && rho < lo);
  const float rho_c = fminf(fmaxf(rho, lo), hi);
  float pg = fmaxf(-adv * rho, -adv * rho_c);
  if (o.clip_dual > 1.0f && adv < 0.0f && pg > -adv * o.clip_dual) {
    pg = -adv * o.clip_dual;
    clipped = true;
  }
  float kl = 0.0f, dkl = 0.0f;
  if (o.kl_coef > 0.0f) {
    const float x = ref - logp;
    if (o.kl_estimator == ECHO_KL_K1) {
      kl = -x;
      dkl = 1.0f;
    } else if (o.kl_estimator == ECHO_KL_K2) {
      kl = 0.5f * x * x;
      dkl = -x;
    } else {
      const float ex = expf(x);
      kl = ex - x - 1.0f;
      dkl = 1.0f - ex;
    }
  }
  const bool ent = o.entropy_coef > 0.0f;
  const float loss = pg + o.kl_coef * kl - (ent ? o.entropy_coef * H : 0.0f);
  const float dl = (clipped ? 0.0f : -adv * rho) + o.kl_coef * dkl;
  const float coef = dl * scale;
  const bool finite = isfinite(lse) && isfinite(logp) && isfinite(rho) && isfinite(loss) && isfinite(coef) &&
                      (!ent || isfinite(H));
  r.logp = logp;
  r.loss = loss;
  r.coef = coef;
  r.ecoef = scale * o.entropy_coef;
  r.flags = (uint8_t)((clipped ? ECHO_FLAG_CLIPPED : 0) | (finite ? 0 : ECHO_FLAG_NONFINITE));
  return r;
}

}  // namespace echo
