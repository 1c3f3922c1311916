// Diagnostic (not part of the library): can a tcgen05 MN-major tf32 operand
// (SWIZZLE_128B_BASE32B) start at a 128-B row that is NOT on a 1024-B swizzle
// boundary, and can TMA land a swizzled box at such a row?  If both follow
// the shared-memory ADDRESS bits, implicit-GEMM convolutions can place
// 32-column atoms at any row pitch (e.g. 33 k-rows per image group) and let
// neighbouring output pixels share one input box at a row offset.
//
// A (M=128, K=8, K-major SW128, built in software) selects row m%8 of the
// K-step; D[m][n] = B[start + m%8][n] shows which rows the MMA read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1610_03618_b200/csrc scripts/swz_test.cu -o build/swz_test -lcuda
#include <cuda.h>
#include <stdio.h>

#include <vector>

#include "tc.cuh"

using namespace lcnn_tc;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int ROWS = 64;  // k-rows in the box

// dst_row: smem row (x 128 B) the TMA box lands at; start_row: first k-row
// the MMA descriptor points at (relative to the 1024-aligned base)
__global__ void __launch_bounds__(128, 1)
    swz_kernel(const __grid_constant__ CUtensorMap tb, float* D, int dst_row, int start_row) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full, done;
  __shared__ uint32_t taddr_s;
  uint8_t* sa = smem;              // A: 128 rows x 128 B (16 KB)
  uint8_t* sb = smem + 16384;      // B region
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // A[m][k] = (k == m % 8), K-major SWIZZLE_128B: chunk c of row m at c ^ (m & 7)
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int m = i / 32, j = i % 32;  // j: float slot in the 128-B row
    reinterpret_cast<float*>(sa + m * 128)[j] = 0.f;
  }
  __syncthreads();
  {
    const int m = threadIdx.x, k = m % 8;
    const int chunk = (k / 4) ^ (m & 7);
    reinterpret_cast<float*>(sa + m * 128 + chunk * 16)[k % 4] = 1.f;
  }
  for (int i = threadIdx.x; i < 160 * 32; i += blockDim.x) reinterpret_cast<float*>(sb)[i] = -1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&full, 1);
      mbar_init(&done, 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<32>(&taddr_s);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = taddr_s;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&full, ROWS * 128);
    tma_load_2d(sb + dst_row * 128, &tb, &full, 0, 0);
    mbar_wait(&full, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_tf32(128, 32, false, true);
    mma_tf32(tmem, smem_desc_sw128(sa, 16, 1024), smem_desc_sw128(sb + start_row * 128, 4096, 512, 1),
             idesc, 0u);
    tc_commit(&done);
  }
  __syncthreads();
  mbar_wait(&done, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
  const int m = warp * 32 + lane;
  for (int j = 0; j < 32; ++j) D[m * 32 + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  // B global: [ROWS k][32 n], value k * 32 + n
  std::vector<float> hb(ROWS * 32);
  for (int k = 0; k < ROWS; ++k)
    for (int n = 0; n < 32; ++n) hb[k * 32 + n] = k * 32.f + n;  // < 2048: exact in tf32
  float *dB, *dD;
  cudaMalloc(&dB, hb.size() * 4);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMemcpy(dB, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tb;
  const cuuint64_t dims[2] = {32, ROWS};
  const cuuint64_t str[1] = {32 * 4};
  const cuuint32_t box[2] = {32, ROWS};
  const cuuint32_t es[2] = {1, 1};
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(swz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int cases[][2] = {{0, 0}, {0, 8}, {0, 1}, {0, 4}, {0, 12}, {0, 16}, {0, 17}, {0, 24},
                          {0, 33}, {0, 41}, {0, 56}, {33, 33}, {33, 41}, {33, 66}, {12, 45},
                          {1, 33}, {45, 57}, {45, 78}, {90, 102}, {90, 135}};
  std::vector<float> hd(128 * 32);
  for (auto& c : cases) {
    const int dst = c[0], start = c[1];
    cudaMemset(dD, 0, 128 * 32 * 4);
    swz_kernel<<<1, 128, 64 * 1024>>>(tb, dD, dst, start);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("dst_row %2d start_row %2d: CUDA error %s\n", dst, start, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hd.data(), dD, hd.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 32; ++n) {
        const int k = start - dst + m % 8;  // box row the MMA should see
        const float want = (k >= 0 && k < ROWS) ? k * 32.f + n : -1.f;
        if (hd[m * 32 + n] != want) ++bad;
      }
    printf("dst_row %2d start_row %2d: %s (%d bad)\n", dst, start, bad ? "MISMATCH" : "ok", bad);
    int shown = 0;
    for (int m = 0; m < 128 && shown < 4; ++m)
      for (int n = 0; n < 32 && shown < 4; ++n) {
        const int k = start - dst + m % 8;
        const float want = (k >= 0 && k < ROWS) ? k * 32.f + n : -1.f;
        if (hd[m * 32 + n] != want) {
          printf("   m%d n%d got %.0f want %.0f\n", m, n, hd[m * 32 + n], want);
          ++shown;
        }
      }
  }
  return 0;
}
