// synth_gen.cu -- GPU twin of synth.logits_rows(): the stand-in for the model's LM-head forward.
//
// TEST / BENCH INFRASTRUCTURE (the seeded input generator).  Holds none of the method's arithmetic: it
// draws Philox4x32-10 counters and writes synthetic logits, bit-identical to the numpy twin in
// synth/__init__.py (same counters, same fp32 operation order with explicit _rn intrinsics, RNE to bf16).
//
// Row r of a micro-batch is packed token t = row0 + r; its global key is
//   T = kept_rollout[slot] * S + (t - kept_offset[slot]),  slot = tok_slot[t]
// so every row's values depend only on (seed, rollout, position) -- not on packing, rank or micro-batch.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint32_t kLabelLogits = 1, kLabelSpike = 3;
constexpr float kLogitScale = 0x1.bb67aep-15f;  // fp32(2 * sqrt(3) / 65536) == synth.LOGIT_SCALE

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

__device__ __forceinline__ float irwin_hall4(uint32_t wa, uint32_t wb) {
  const int32_t s = (int32_t)(wa & 0xFFFFu) + (int32_t)(wa >> 16) + (int32_t)(wb & 0xFFFFu) + (int32_t)(wb >> 16) -
                    131070;
  return __fmul_rn((float)s, kLogitScale);
}

template <bool BF16>
__global__ void __launch_bounds__(256) fill_logits_kernel(uint8_t* logits, int64_t n_rows, int32_t V, int64_t ld,
                                                          int64_t row0, const int32_t* __restrict__ tok_slot,
                                                          const int32_t* __restrict__ tok_action,
                                                          const int32_t* __restrict__ kept_rollout,
                                                          const int64_t* __restrict__ kept_offset, int32_t S,
                                                          uint32_t seed) {
  const int32_t npairs = (V + 1) / 2;
  for (int64_t row = blockIdx.y; row < n_rows; row += gridDim.y) {
    const int64_t t = row0 + row;
    const int32_t slot = tok_slot[t];
    const int64_t T = (int64_t)kept_rollout[slot] * S + (t - kept_offset[slot]);
    const uint32_t tlo = (uint32_t)T, thi = (uint32_t)((uint64_t)T >> 32);
    const int32_t a = tok_action[t];
    const U4 ws = philox4x32_10(U4{tlo, thi, 0u, 0u}, seed, kLabelSpike);
    const float u = __fmul_rn((float)(ws.x >> 8), 0x1p-24f);
    const float spike = __fadd_rn(8.0f, __fmul_rn(12.0f, u));
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += gridDim.x * blockDim.x) {
      const U4 w = philox4x32_10(U4{(uint32_t)q, tlo, thi, 0u}, seed, kLabelLogits);
      float z0 = irwin_hall4(w.x, w.y), z1 = irwin_hall4(w.z, w.w);
      const int32_t c = 2 * q;
      if (c == a) z0 = __fadd_rn(z0, spike);
      if (c + 1 == a) z1 = __fadd_rn(z1, spike);
      if (BF16) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(logits + row * ld * 2);
        if (c + 1 < V) {
          *reinterpret_cast<__nv_bfloat162*>(dst + c) = __floats2bfloat162_rn(z0, z1);
        } else {
          dst[c] = __float2bfloat16_rn(z0);
        }
      } else {
        float* dst = reinterpret_cast<float*>(logits + row * ld * 4);
        dst[c] = z0;
        if (c + 1 < V) dst[c + 1] = z1;
      }
    }
  }
}

}  // namespace

extern "C" {

// dtype: 0 = fp32, 1 = bf16.  All pointers are device pointers; returns a cudaError_t value.
__attribute__((visibility("default"))) int synth_fill_logits(void* logits, int32_t dtype, int64_t n_rows, int32_t V,
                                                             int64_t ld, int64_t row0, const int32_t* tok_slot,
                                                             const int32_t* tok_action, const int32_t* kept_rollout,
                                                             const int64_t* kept_offset, int32_t S, uint32_t seed,
                                                             void* stream) {
  if (n_rows <= 0) return 0;
  const int32_t npairs = (V + 1) / 2;
  dim3 grid((unsigned)((npairs + 255) / 256), (unsigned)(n_rows < 65535 ? n_rows : 65535));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == 1)
    fill_logits_kernel<true><<<grid, 256, 0, s>>>(static_cast<uint8_t*>(logits), n_rows, V, ld, row0, tok_slot,
                                                  tok_action, kept_rollout, kept_offset, S, seed);
  else
    fill_logits_kernel<false><<<grid, 256, 0, s>>>(static_cast<uint8_t*>(logits), n_rows, V, ld, row0, tok_slot,
                                                   tok_action, kept_rollout, kept_offset, S, seed);
  return (int)cudaGetLastError();
}

}  // extern "C"
