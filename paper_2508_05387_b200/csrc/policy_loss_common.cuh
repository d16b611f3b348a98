// policy_loss_common.cuh -- per-row helpers shared by the fused policy-loss kernels.
#pragma once

#include <cuda_bf16.h>

#include "echo_common.cuh"
#include "echo_internal.h"

namespace echo {

// Phase timestamps for tools/trace_kernel.py (compiled in only with -DECHO_TRACE, i.e. libecho_trace.so).
#ifdef ECHO_TRACE
#define ECHO_TRACE_MARK(p, it, k)                                                                   \
  do {                                                                                               \
    if (threadIdx.x == 0 && (p).trace && (it) < (uint32_t)(p).trace_rows && blockIdx.x < 64)         \
      (p).trace[((size_t)blockIdx.x * (p).trace_rows + (it)) * 16 + (k)] = clock64();                \
  } while (0)
#else
#define ECHO_TRACE_MARK(p, it, k) \
  do {                            \
  } while (0)
#endif

// ====================================================================== shared per-row helpers
struct RowMeta {
  float old, ref, adv, w;  // w: per-token loss weight (1 when the 1 / N_global scale applies)
};
ECHO_DEVINL RowMeta load_meta(const LossParams& p, int64_t row) {
  RowMeta m;
  m.old = p.tok_old[row];
  m.ref = (p.kl_coef > 0.0f) ? p.tok_ref[row] : 0.0f;
  m.adv = p.tok_adv ? p.tok_adv[row] : p.adv_slot[p.tok_slot[row]];
  m.w = p.tok_weight ? p.tok_weight[row] : 1.0f;
  return m;
}
ECHO_DEVINL LossOpts loss_opts(const LossParams& p) {
  return LossOpts{p.clip_low, p.clip_high, p.clip_dual, p.kl_coef, p.kl_estimator, p.entropy_coef};
}
// grad_scale / N_global, or grad_scale alone when per-token weights carry the normalisation
ECHO_DEVINL float base_scale(const LossParams& p) {
  return p.tok_weight ? p.grad_scale : (float)((double)p.grad_scale / *p.n_global);
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

// Same with the entropy accumulator t = sum x e^{x - m} (masked -inf entries contribute 0).
template <int N>
ECHO_DEVINL void online_update3(MaxSum& acc, float& t, const float (&x)[N]) {
  float cm = x[0];
#pragma unroll
  for (int e = 1; e < N; ++e) cm = fmaxf(cm, x[e]);
  if (cm > acc.m) {
    const float f = ex2((acc.m - cm) * kLog2e);
    acc.s = acc.s * f;
    t = t * f;
    acc.m = cm;
  }
  const float mb = (acc.m == -INFINITY) ? 0.0f : acc.m * kLog2e;
  float ss = 0.0f, tt = 0.0f;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float xe = fmaxf(x[e], -1.0e30f);
    const float ev = ex2(fmaf(xe, kLog2e, -mb));
    ss += ev;
    tt = fmaf(ev, xe, tt);
  }
  acc.s += ss;
  t += tt;
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

// With the entropy term: d_v = c (delta_{v,a} - p_v) + e p_v (z_v - lse + H); masked -inf entries get the plain
// c (delta - p) = 0.
template <int N>
ECHO_DEVINL void grad_values_ent(float (&x)[N], int32_t col0, int32_t a, float coef, float lse_l2e, float lse, float H,
                                 float ecoef) {
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float p = ex2(fmaf(x[e], kLog2e, -lse_l2e));
    float d = (col0 + e == a) ? fmaf(-coef, p, coef) : -coef * p;
    if (x[e] != -INFINITY) d = fmaf(ecoef * p, x[e] - lse + H, d);
    x[e] = d;
  }
}

// Set the bf16 lanes >= nkeep of an 8-lane vector to -inf.
ECHO_DEVINL uint4 mask_tail(uint4 w, int nkeep) {
  uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (e >= nkeep) x[e >> 1] = (e & 1) ? ((x[e >> 1] & 0x0000FFFFu) | 0xFF800000u) : ((x[e >> 1] & 0xFFFF0000u) | 0x0000FF80u);
  return make_uint4(x[0], x[1], x[2], x[3]);
}

// Store the first n (< 8) bf16 lanes of a packed vector.
ECHO_DEVINL void store_partial8(__nv_bfloat16* dd, const uint4& o, int n) {
  const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (e < n) dd[e] = __ushort_as_bfloat16((unsigned short)((e & 1) ? (ow[e >> 1] >> 16) : (ow[e >> 1] & 0xFFFFu)));
}

}  // namespace echo
