// Write-pattern microbenchmark (sm_100a): VGG conv1_1's output stream.  The
// ROW row-pair kernel writes, per tile, 2 output rows x 64 channels x one
// 1 KB run (2 pixels x 128 images, CHWN) -- 128 runs a channel plane
// (224*224*128*4 = 25.7 MB) apart; 12544 tiles round-robin over 148 CTAs.
// Is that pattern itself slower than a contiguous write of the same 1.6 GB?
//   A: lane = channel, each lane stores its 1 KB run as 64 float4 (per-lane)
//   B: the warp stores one run at a time, 32 lanes x 2 float4 (coalesced)
//   C: contiguous: the same bytes as one linear stream (grid-stride float4)
//   D: the kernel's chunk order: per (pixel, 32-image chunk) 32 channels x one 128 B line,
//      4 channels x 128 B per instruction (the epilogue's coalesced per-chunk stores)
//   E: per pixel, 32 channels x one 512 B run (all 128 images), 1 channel x 512 B per instruction
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/store_pattern_bench scripts/store_pattern_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr uint32_t H = 224, W = 224, N = 128, C = 64;
constexpr uint64_t PLANE = uint64_t(H) * W * N;  // floats
constexpr uint32_t TILES = (H / 2) * (W / 2);

// 4 warps (the epilogue warps) per CTA; warp q holds 32 channels of one row
template <int MODE>
__global__ void __launch_bounds__(128) tiles_kernel(float* __restrict__ y, float v) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c0 = (q & 1) * 32, dr = q >> 1;
  const float4 f = make_float4(v, v, v, v);
  for (uint32_t t = blockIdx.x; t < TILES; t += gridDim.x) {
    const uint32_t pr = t / (W / 2), wp = t % (W / 2);
    const uint32_t h = 2 * pr + dr, w0 = 2 * wp;
    if (MODE == 0) {
      float4* dst = reinterpret_cast<float4*>(y + ((uint64_t(c0 + lane) * H + h) * W + w0) * N);
#pragma unroll 8
      for (int j = 0; j < 64; ++j) dst[j] = f;
    } else if (MODE == 2) {
      for (uint32_t px = 0; px < 2; ++px)
        for (uint32_t ch = 0; ch < 4; ++ch)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t c = 4 * k + (lane >> 3), j = lane & 7;
            float4* dst = reinterpret_cast<float4*>(
                y + ((uint64_t(c0 + c) * H + h) * W + w0 + px) * N + ch * 32);
            dst[j] = f;
          }
    } else if (MODE == 3) {
      for (uint32_t px = 0; px < 2; ++px)
        for (int c = 0; c < 32; ++c) {
          float4* dst = reinterpret_cast<float4*>(y + ((uint64_t(c0 + c) * H + h) * W + w0 + px) * N);
          dst[lane] = f;
        }
    } else {
      for (int c = 0; c < 32; ++c) {
        float4* dst = reinterpret_cast<float4*>(y + ((uint64_t(c0 + c) * H + h) * W + w0) * N);
        dst[lane] = f;
        dst[lane + 32] = f;
      }
    }
  }
}

__global__ void linear_kernel(float4* __restrict__ y, uint64_t n4, float v) {
  const float4 f = make_float4(v, v, v, v);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x)
    y[i] = f;
}

int main() {
  const uint64_t bytes = PLANE * C * 4;
  float* y;
  CK(cudaMalloc(&y, bytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int K = 20;
  auto report = [&](const char* name, float ms) {
    printf("%-44s %8.1f us  %7.1f GB/s\n", name, ms * 1e3 / K, bytes / (ms * 1e-3 / K) / 1e9);
  };
  for (int rep = 0; rep < 2; ++rep) {
    for (int g : {148, 296}) {
      float ms;
      for (int i = 0; i < 3; ++i) tiles_kernel<0><<<g, 128>>>(y, 1.f);
      CK(cudaEventRecord(a));
      for (int i = 0; i < K; ++i) tiles_kernel<0><<<g, 128>>>(y, float(i));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      report(g == 148 ? "A per-lane 1 KB runs, 148 CTAs" : "A per-lane 1 KB runs, 296 CTAs", ms);
      for (int i = 0; i < 3; ++i) tiles_kernel<1><<<g, 128>>>(y, 1.f);
      CK(cudaEventRecord(a));
      for (int i = 0; i < K; ++i) tiles_kernel<1><<<g, 128>>>(y, float(i));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      report(g == 148 ? "B coalesced 1 KB runs, 148 CTAs" : "B coalesced 1 KB runs, 296 CTAs", ms);
    }
    {
      float ms;
      for (int i = 0; i < 3; ++i) tiles_kernel<2><<<148, 128>>>(y, 1.f);
      CK(cudaEventRecord(a));
      for (int i = 0; i < K; ++i) tiles_kernel<2><<<148, 128>>>(y, float(i));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      report("D kernel order, 128 B lines, 148 CTAs", ms);
      for (int i = 0; i < 3; ++i) tiles_kernel<3><<<148, 128>>>(y, 1.f);
      CK(cudaEventRecord(a));
      for (int i = 0; i < K; ++i) tiles_kernel<3><<<148, 128>>>(y, float(i));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      report("E per pixel 512 B runs, 148 CTAs", ms);
    }
    float ms;
    for (int i = 0; i < 3; ++i) linear_kernel<<<148 * 8, 512>>>(reinterpret_cast<float4*>(y), bytes / 16, 1.f);
    CK(cudaEventRecord(a));
    for (int i = 0; i < K; ++i) linear_kernel<<<148 * 8, 512>>>(reinterpret_cast<float4*>(y), bytes / 16, float(i));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    report("C contiguous stream", ms);
  }
  CK(cudaGetLastError());
  return 0;
}
