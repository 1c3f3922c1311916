// DRAM-cold streaming microbenchmark (sm_100a): how long one launch takes to
// read R contiguous bytes (the packed fc weights: 151 MB for AlexNet fc6,
// 67 MB for fc7) when every CTA streams its own contiguous range through a
// shared-memory ring of cp.async.bulk copies (the fc producer's pattern), and
// the same bytes read by a plain 128-bit-load grid (sum into one word).  The
// source rotates over enough copies (> 4x L2) that each launch reads HBM.
// t(R) over two sizes gives the per-launch overhead (intercept) and the
// streaming rate (slope): what an fc kernel can reach at best.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_bench scripts/stream_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one CTA per SM; thread 0 issues bulk copies of `slot` bytes into a ring of
// `stages` slots, thread 32 waits for each slot and frees it at once
__global__ void __launch_bounds__(64, 1)
    ring_kernel(const uint8_t* __restrict__ src, uint64_t bytes, uint32_t slot, uint32_t stages,
                uint64_t* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  __shared__ uint64_t full[16], empty[16];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint64_t per = (bytes / gridDim.x + slot - 1) / slot * slot;
  const uint64_t lo = per * blockIdx.x;
  const uint64_t hi = lo + per < bytes ? lo + per : bytes;
  const uint32_t n = lo < hi ? static_cast<uint32_t>((hi - lo + slot - 1) / slot) : 0;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % stages, ph = (i / stages) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
              sa(&empty[s])),
          "r"(ph ^ 1));
      const uint64_t off = lo + static_cast<uint64_t>(i) * slot;
      const uint32_t b = static_cast<uint32_t>(hi - off < slot ? hi - off : slot);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(b));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sa(smem + s * slot)),
          "l"(src + off), "r"(b), "r"(sa(&full[s]))
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    uint64_t acc = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % stages, ph = (i / stages) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
              sa(&full[s])),
          "r"(ph));
      acc += smem[s * slot];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])));
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

__global__ void __launch_bounds__(512) ldg_kernel(const uint4* __restrict__ src, uint64_t n16,
                                                  uint64_t* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * 512ull + threadIdx.x; i < n16; i += gridDim.x * 512ull) {
    const uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const uint64_t sizes[2] = {67108864ull, 150994944ull};  // fc7, fc6 weights
  const int copies = 4;
  uint8_t* buf;
  uint64_t* sink;
  CK(cudaMalloc(&buf, sizes[1] * copies));
  CK(cudaMemset(buf, 1, sizes[1] * copies));
  CK(cudaMalloc(&sink, 8));
  CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 231424));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct R {
    uint32_t slot, stages;
  } rings[] = {{32768, 4}, {32768, 6}, {16384, 8}, {16384, 12}, {65536, 3}, {49152, 4}, {8192, 16}};
  const int K = 40;
  for (int z = 0; z < 2; ++z) {
    const uint64_t bytes = sizes[z];
    for (const R& r : rings) {
      for (int g : {148, 296}) {
        const size_t smem = static_cast<size_t>(r.slot) * r.stages + 1024;
        if (g == 296 && smem > 110000) continue;
        for (int w = 0; w < 4; ++w)
          ring_kernel<<<g, 64, smem>>>(buf + (w % copies) * sizes[1], bytes, r.slot, r.stages, sink);
        CK(cudaEventRecord(a));
        for (int i = 0; i < K; ++i)
          ring_kernel<<<g, 64, smem>>>(buf + (i % copies) * sizes[1], bytes, r.slot, r.stages, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double us = ms * 1e3 / K;
        printf("ring  %6.1f MB  slot %6u x %2u  grid %3d  %7.2f us  %7.1f GB/s\n", bytes / 1048576.0,
               r.slot, r.stages, g, us, bytes / us / 1e3);
      }
    }
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      for (int w = 0; w < 4; ++w)
        ldg_kernel<<<g, 512>>>(reinterpret_cast<const uint4*>(buf + (w % copies) * sizes[1]), bytes / 16, sink);
      CK(cudaEventRecord(a));
      for (int i = 0; i < K; ++i)
        ldg_kernel<<<g, 512>>>(reinterpret_cast<const uint4*>(buf + (i % copies) * sizes[1]), bytes / 16, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double us = ms * 1e3 / K;
      printf("ldg   %6.1f MB  grid %5d x 512            %7.2f us  %7.1f GB/s\n", bytes / 1048576.0, g, us,
             bytes / us / 1e3);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
