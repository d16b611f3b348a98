// membench.cu -- memory-pipeline microbenchmarks for the fused policy-loss design (diagnostic tool, not product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/membench tools/membench.cu
//
// Streams a [rows x V] bf16 buffer in the shapes the kernels use and reports GB/s of algorithmic traffic:
//   mode 0: TMA ring read only (1 CTA/SM, producer warp + 15 consumer warps LDS + release)
//   mode 1: TMA ring read + STG.128 write-back of the same data in place (no math)
//   mode 2: plain LDG.128 / STG.128 in-place stream (grid-stride, 8 CTAs/SM x 256 thr, 4 vectors in flight)
//   mode 3: mode 1 with the CTA pair (2 CTAs per row) geometry and a per-row cluster exchange (no math)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define DEVINL __device__ __forceinline__
DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
DEVINL void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
DEVINL void mbar_arrive(uint32_t b) {
  asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(b) : "memory");
}
DEVINL void mbar_expect(uint32_t b, uint32_t tx) {
  asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(b), "r"(tx) : "memory");
}
DEVINL void mbar_wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok)
                 : "r"(b), "r"(ph)
                 : "memory");
}
DEVINL uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
DEVINL void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
               "l"(src), "r"(n), "r"(bar), "l"(pol)
               : "memory");
}
DEVINL uint4 lds(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
DEVINL void stg(void* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
DEVINL void stg_plain(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
DEVINL uint4 ldg_plain(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
DEVINL uint4 ldg(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

constexpr int CW = 15, CT = CW * 32, NT = CT + 32, CH = CT * 16, RING = 27;

template <bool kWrite, bool kPlainStore = false>
__global__ void __launch_bounds__(NT, 1) ring_kernel(uint8_t* buf, int64_t rows, int64_t row_bytes, int splits) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + RING * CH);
  uint64_t* empty = full + RING;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // work units: (row, part) with part in [0, splits)
  const int64_t part_bytes = row_bytes / splits;
  const int nch = (int)((part_bytes + CH - 1) / CH);
  const int64_t units = rows * splits;
  if (tid == 0) {
    for (int i = 0; i < RING; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint64_t pol = pol_first();
  if (warp == CW) {
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint8_t* src = buf + (u / splits) * row_bytes + (u % splits) * part_bytes;
        for (int c = 0; c < nch; ++c) {
          mbar_wait(smem_u32(&empty[slot]), ph ^ 1);
          const uint32_t nb = (uint32_t)min((int64_t)CH, part_bytes - (int64_t)c * CH);
          mbar_expect(smem_u32(&full[slot]), nb);
          bulk(smem_u32(sm + slot * CH), src + (int64_t)c * CH, nb, smem_u32(&full[slot]), pol);
          if (++slot == RING) { slot = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  uint32_t slot = 0, ph = 0;
  uint32_t acc = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    uint8_t* dst = buf + (u / splits) * row_bytes + (u % splits) * part_bytes;
    for (int c = 0; c < nch; ++c) {
      mbar_wait(smem_u32(&full[slot]), ph);
      const uint4 v = lds(smem_u32(sm + slot * CH + tid * 16));
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      if (++slot == RING) { slot = 0; ph ^= 1; }
      const int64_t off = (int64_t)c * CH + tid * 16;
      if (kWrite) {
        if (off < part_bytes) {
          if (kPlainStore) stg_plain(dst + off, v);
          else stg(dst + off, v, pol);
        }
      } else {
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
  }
  if (acc == 0x12345678u) buf[0] = 1;
}

__global__ void __launch_bounds__(256) stream_kernel(uint8_t* buf, int64_t n16) {
  const uint64_t pol = pol_first();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n16) v[u] = ldg(buf + (i + u * stride) * 16, pol);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n16) {
        v[u].x ^= 0x80008000u;
        stg(buf + (i + u * stride) * 16, v[u], pol);
      }
  }
}

// torch-like tiles: block b owns the contiguous tile [b T, (b+1) T) of 16-byte vectors, T = 256 x kU; all kU loads
// are issued before the stores (kPersist: grid-stride over tiles with one block per SM slot)
template <int kU, bool kPol, bool kPersist>
__global__ void __launch_bounds__(256) tile_kernel(uint8_t* buf, int64_t n16) {
  const uint64_t pol = pol_first();
  const int64_t ntiles = (n16 + 256 * kU - 1) / (256 * kU);
  for (int64_t t = blockIdx.x; t < ntiles; t += kPersist ? gridDim.x : ntiles) {
    const int64_t base = t * 256 * kU + threadIdx.x;
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (base + u * 256 < n16) v[u] = kPol ? ldg(buf + (base + u * 256) * 16, pol) : ldg_plain(buf + (base + u * 256) * 16);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (base + u * 256 < n16) {
        v[u].x ^= 0x80008000u;
        if (kPol) stg(buf + (base + u * 256) * 16, v[u], pol);
        else stg_plain(buf + (base + u * 256) * 16, v[u]);
      }
  }
}

// persistent, but tiles handed out in order by a global atomic counter (keeps the in-flight window compact)
template <int kU>
__global__ void __launch_bounds__(256) tile_atomic_kernel(uint8_t* buf, int64_t n16, unsigned long long* counter) {
  __shared__ int64_t next;
  const int64_t ntiles = (n16 + 256 * kU - 1) / (256 * kU);
  for (;;) {
    if (threadIdx.x == 0) next = (int64_t)atomicAdd(counter, 1ull);
    __syncthreads();
    const int64_t t = next;
    __syncthreads();
    if (t >= ntiles) break;
    const int64_t base = t * 256 * kU + threadIdx.x;
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (base + u * 256 < n16) v[u] = ldg_plain(buf + (base + u * 256) * 16);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (base + u * 256 < n16) {
        v[u].x ^= 0x80008000u;
        stg_plain(buf + (base + u * 256) * 16, v[u]);
      }
  }
}

// ring read + write with rows handed out by an atomic counter (one producer lane grabs the next row, the consumer
// warps learn it through a shared-memory slot per ring row)
__global__ void __launch_bounds__(NT, 1) ring_atomic_kernel(uint8_t* buf, int64_t rows, int64_t row_bytes,
                                                            unsigned long long* counter) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + RING * CH);
  uint64_t* empty = full + RING;
  int64_t* rowq = (int64_t*)(empty + RING);  // row of each ring slot
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (int)((row_bytes + CH - 1) / CH);
  if (tid == 0) {
    for (int i = 0; i < RING; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint64_t pol = pol_first();
  if (warp == CW) {
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      for (;;) {
        const int64_t u = (int64_t)atomicAdd(counter, 1ull);
        const bool done = u >= rows;
        const uint8_t* src = buf + u * row_bytes;
        for (int c = 0; c < (done ? 1 : nch); ++c) {
          mbar_wait(smem_u32(&empty[slot]), ph ^ 1);
          rowq[slot] = done ? -1 : u;
          if (done) {
            mbar_arrive(smem_u32(&full[slot]));
          } else {
            const uint32_t nb = (uint32_t)min((int64_t)CH, row_bytes - (int64_t)c * CH);
            mbar_expect(smem_u32(&full[slot]), nb);
            bulk(smem_u32(sm + slot * CH), src + (int64_t)c * CH, nb, smem_u32(&full[slot]), pol);
          }
          if (++slot == RING) { slot = 0; ph ^= 1; }
        }
        if (done) break;
      }
    }
    return;
  }
  uint32_t slot = 0, ph = 0;
  for (;;) {
    mbar_wait(smem_u32(&full[slot]), ph);
    const int64_t u = rowq[slot];
    if (u < 0) break;
    uint8_t* dst = buf + u * row_bytes;
    for (int c = 0; c < nch; ++c) {
      if (c > 0) mbar_wait(smem_u32(&full[slot]), ph);
      const uint4 v = lds(smem_u32(sm + slot * CH + tid * 16));
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      if (++slot == RING) { slot = 0; ph ^= 1; }
      const int64_t off = (int64_t)c * CH + tid * 16;
      if (off < row_bytes) stg(dst + off, v, pol);
    }
  }
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 32768;
  const int64_t V = argc > 2 ? atoll(argv[2]) : 151936;
  const int64_t row_bytes = V * 2;
  uint8_t* buf;
  const size_t bytes = (size_t)rows * row_bytes;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = RING * CH + 2 * RING * 8;
  cudaFuncSetAttribute(ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(ring_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(ring_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn, double traffic) {
    for (int w = 0; w < 2; ++w) fn();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("{\"mode\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n", name, ms, traffic / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int splits : {1, 2, 4}) {
    char n0[64], n1[64];
    snprintf(n0, 64, "ring_read_split%d", splits);
    snprintf(n1, 64, "ring_read_write_split%d", splits);
    run(n0, [&] { ring_kernel<false><<<sms, NT, smem>>>(buf, rows, row_bytes, splits); }, (double)bytes);
    run(n1, [&] { ring_kernel<true><<<sms, NT, smem>>>(buf, rows, row_bytes, splits); }, 2.0 * bytes);
  }
  run("ring_read_write_split1_plainstore", [&] { ring_kernel<true, true><<<sms, NT, smem>>>(buf, rows, row_bytes, 1); },
      2.0 * bytes);
  const int64_t n16 = (int64_t)(bytes / 16);
  const int64_t nt4 = (n16 + 1023) / 1024, nt8 = (n16 + 2047) / 2048;
  unsigned long long* counter;
  cudaMalloc(&counter, 8);
  run("tile4_atomic_persist8", [&] {
    cudaMemsetAsync(counter, 0, 8);
    tile_atomic_kernel<4><<<sms * 8, 256>>>(buf, n16, counter);
  }, 2.0 * bytes);
  cudaFuncSetAttribute(ring_atomic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + RING * 8));
  run("ring_read_write_atomic_rows", [&] {
    cudaMemsetAsync(counter, 0, 8);
    ring_atomic_kernel<<<sms, NT, smem + RING * 8>>>(buf, rows, row_bytes, counter);
  }, 2.0 * bytes);
  run("tile4_plain", [&] { tile_kernel<4, false, false><<<(unsigned)nt4, 256>>>(buf, n16); }, 2.0 * bytes);
  run("tile4_evict_first", [&] { tile_kernel<4, true, false><<<(unsigned)nt4, 256>>>(buf, n16); }, 2.0 * bytes);
  run("tile8_plain", [&] { tile_kernel<8, false, false><<<(unsigned)nt8, 256>>>(buf, n16); }, 2.0 * bytes);
  run("tile4_plain_persist8", [&] { tile_kernel<4, false, true><<<sms * 8, 256>>>(buf, n16); }, 2.0 * bytes);
  run("tile4_evict_first_persist8", [&] { tile_kernel<4, true, true><<<sms * 8, 256>>>(buf, n16); }, 2.0 * bytes);
  run("tile8_plain_persist4", [&] { tile_kernel<8, false, true><<<sms * 4, 256>>>(buf, n16); }, 2.0 * bytes);
  for (int per_sm : {2, 4, 8}) {
    char n2[64];
    snprintf(n2, 64, "ldg_stg_stream_%dcta", per_sm);
    run(n2, [&] { stream_kernel<<<sms * per_sm, 256>>>(buf, (int64_t)(bytes / 16)); }, 2.0 * bytes);
  }
  cudaFree(buf);
  return 0;
}
