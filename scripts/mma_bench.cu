// tcgen05 kind::tf32 issue-rate microbenchmark (sm_100a): cycles per MMA
// instruction (M = 128, K = 8) for the operand layouts and N widths the
// implicit-GEMM convolutions use.  One CTA per SM, one thread issues `iters`
// groups of `per` MMAs on fixed shared-memory operands, committing each group
// to an mbarrier (as the pipeline does), then waits for the last commit.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_bench scripts/mma_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_1610_03618_b200/csrc/tc.cuh"

using namespace lcnn_tc;

struct Cfg {
  uint32_t idesc;
  uint32_t a_layout, a_lbo, a_sbo, a_step;  // A descriptor: layout, LBO, SBO, K-step advance
  uint32_t b_layout, b_lbo, b_sbo, b_step;
  int per, iters;
  int nacc = 1;  // independent accumulators the MMAs rotate over
  int fused = 0;  // 1: the 4 MMAs of a group in one asm block (descriptor adds in PTX)
};

__global__ void __launch_bounds__(128, 1) mma_kernel(const __grid_constant__ Cfg c, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t taddr;
  for (uint32_t i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<512>(&taddr);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint8_t* sa = smem;
    const uint8_t* sb = smem + 48 * 1024;
    // descriptors and accumulator addresses hoisted out of the loop, so the
    // issue loop is just the MMAs (the first version of this bench rebuilt
    // them per MMA and measured the single-thread issue cost, ~150 cycles)
    uint64_t da[4], db[4];
    uint32_t dt[4];
    const uint32_t ncol = ((c.idesc >> 17) & 0x3F) * 8;
    for (int k = 0; k < 4; ++k) {
      da[k] = smem_desc_sw128(sa + k * c.a_step, c.a_lbo, c.a_sbo, c.a_layout);
      db[k] = smem_desc_sw128(sb + k * c.b_step, c.b_lbo, c.b_sbo, c.b_layout);
      dt[k] = taddr + (k % c.nacc) * ncol;
    }
    for (int k = 0; k < 4; ++k) mma_tf32(dt[k], da[k], db[k], c.idesc, 0u);
    const long long t0 = clock64();
    for (int it = 0; it < c.iters; ++it) {
      // a group may start once the group 4 back has completed (4-slot ring)
      if (it >= 4) mbar_wait(&bar[it & 3], ((it >> 2) - 1) & 1);
      if (c.fused) {
        asm volatile(
            "{\n.reg .b64 a1, a2, a3, b1, b2, b3;\n"
            "add.s64 a1, %1, %3;\nadd.s64 a2, a1, %3;\nadd.s64 a3, a2, %3;\n"
            "add.s64 b1, %2, %4;\nadd.s64 b2, b1, %4;\nadd.s64 b3, b2, %4;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %5, 1;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %5, 1;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %5, 1;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %5, 1;\n}\n" ::"r"(dt[0]),
            "l"(da[0]), "l"(db[0]), "l"(uint64_t(c.a_step >> 4)), "l"(uint64_t(c.b_step >> 4)),
            "r"(c.idesc)
            : "memory");
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_tf32(dt[k], da[k], db[k], c.idesc, 1u);
      }
      tc_commit(&bar[it & 3]);
    }
    for (int it = c.iters - 4; it < c.iters; ++it) mbar_wait(&bar[it & 3], (it >> 2) & 1);
    const long long t1 = clock64();
    cyc[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(taddr);
  }
}

static void run(const char* name, Cfg c) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 97 * 1024;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<<<148, 128, smem>>>(c, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_kernel<<<148, 128, smem>>>(c, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double n_mma = double(c.iters) * 4;
  const uint32_t N = ((c.idesc >> 17) & 0x3F) * 8;
  const uint32_t M = ((c.idesc >> 24) & 0x1F) * 16;
  const double tflops = 148.0 * n_mma * 2 * M * N * 8 / (ms * 1e9);
  printf("%-40s M=%3u acc=%d N=%3u  %7.1f cyc/MMA  %7.1f TF/s  %s\n", name, M, c.nacc, N, double(h[0]) / n_mma, tflops,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int iters = 4000;
  if (argc > 1) {  // M = 64 (half the tensor rows): does it cost half an M = 128 MMA?
    for (uint32_t N : {64u, 128u, 192u, 256u}) {
      Cfg k{idesc_tf32(64, N, false, true), 2, 16, 1024, 32, 1, 4096, 512, 1024, 4, iters};
      run("M64 A K-sw128 B MN-sw128_32b", k);
      Cfg c{idesc_tf32(128, N, false, true), 2, 16, 1024, 32, 1, 4096, 512, 1024, 4, iters};
      run("M128 A K-sw128 B MN-sw128_32b", c);
    }
    return 0;
  }
  for (uint32_t N : {32u, 64u, 96u, 128u, 192u, 256u}) {
    // A MN-major SW128_32B (the CHWN input operand), B K-major SW128 (packed filters)
    Cfg c{idesc_tf32(128, N, true, false), 1, 4096, 512, 1024, 2, 16, 1024, 32, 4, iters};
    run("A MN-sw128_32b  B K-sw128", c);
    // B K-major no-swizzle core matrices (ROW mode filter image)
    Cfg r{idesc_tf32(128, N, true, false), 1, 5120, 512, 1024, 0, N * 16, 128, 2 * N * 16, 5, iters};
    run("A MN-sw128_32b  B K-none (ROW)", r);
    // both K-major SW128 (plain GEMM A / NCHW conv)
    Cfg g{idesc_tf32(128, N, false, false), 2, 16, 1024, 32, 2, 16, 1024, 32, 4, iters};
    run("A K-sw128       B K-sw128", g);
    // A K-major, B MN-major (fc GEMM)
    Cfg f{idesc_tf32(128, N, false, true), 2, 16, 1024, 32, 1, 4096, 512, 1024, 4, iters};
    run("A K-sw128       B MN-sw128_32b", f);
  }
  for (uint32_t N : {32u, 64u, 96u, 128u, 192u, 256u}) {
    Cfg c{idesc_tf32(128, N, true, false), 1, 4096, 512, 1024, 2, 16, 1024, 32, 4, iters, 1, 1};
    run("fused-asm A MN-sw128_32b B K-sw128", c);
  }
  for (uint32_t N : {32u, 64u, 96u, 128u, 192u, 256u}) {
    Cfg c{idesc_tf32(128, N, true, false), 1, 4096, 512, 1024, 2, 16, 1024, 32, 4, iters, 1, 1};
    run("fused-asm A MN-sw128_32b B K-sw128", c);
  }
  // conv1 SHARE operands: A = filters K-major SWIZZLE_NONE core matrices
  // (bn = 96 rows), B = input MN-major SW128_32B with overlapping atoms
  // (LBO = 12 rows = 1536 B)
  {
    Cfg s{idesc_tf32(128, 256, false, true), 0, 1536, 128, 3072, 1, 1536, 512, 1024, 4, iters};
    run("SHARE A K-none B MN-overlap(1536)", s);
    Cfg t{idesc_tf32(128, 256, false, true), 0, 1536, 128, 3072, 1, 4096, 512, 1024, 4, iters};
    run("SHARE A K-none B MN lbo4096", t);
    Cfg u{idesc_tf32(128, 256, false, true), 2, 16, 1024, 32, 1, 1536, 512, 1024, 4, iters};
    run("A K-sw128 B MN-overlap(1536)", u);
    Cfg v{idesc_tf32(128, 256, false, true), 0, 2048, 128, 4096, 1, 4096, 512, 1024, 4, iters};
    run("A K-none(bn=128) B MN lbo4096", v);
  }
  // independent accumulators: is ~150 cycles a per-MMA latency of one chain?
  for (uint32_t N : {64u, 96u, 128u, 256u})
    for (int nacc : {2, 4}) {
      if (N * nacc > 512) continue;
      Cfg c{idesc_tf32(128, N, true, false), 1, 4096, 512, 1024, 2, 16, 1024, 32, 4, iters, nacc};
      run("A MN-sw128_32b  B K-sw128", c);
    }
  return 0;
}
