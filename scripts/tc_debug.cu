// Standalone diagnostic for the tcgen05 GEMM building blocks (not part of
// the library): 128x128x128 tf32 GEMM with A = I and an encoded B, dumping
// the TMA-filled shared memory so the swizzled layouts and the MMA operand
// descriptors can be checked separately.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_1610_03618_b200/csrc scripts/tc_debug.cu -o build/tc_debug
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "tc.cuh"

using namespace lcnn_tc;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int M = 128, N = 128, K = 128, BK = 32;


__global__ void __launch_bounds__(192, 1)
    dbg_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
               float* C, float* dump, int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[4], tfull;
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < 4; ++s) mbar_init(&full[s], 1);
      mbar_init(&tfull, 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<128>(&taddr_s);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = taddr_s;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < K / BK; ++kb) {
      uint8_t* sa = smem + kb * 32768;
      uint8_t* sb = sa + 16384;
      mbar_arrive_expect_tx(&full[kb], 32768);
      tma_load_2d(sa, &ta, &full[kb], kb * BK, 0);
      if (variant == 2) tma_load_2d(sb, &tb, &full[kb], kb * BK, 0);
      else
        for (int j = 0; j < 4; ++j) tma_load_2d(sb + j * 4096, &tb, &full[kb], 32 * j, kb * BK);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_tf32(128, 128, false, variant != 2);
    for (int kb = 0; kb < K / BK; ++kb) {
      mbar_wait(&full[kb], 0);
      tc_fence_after();
      const uint8_t* sa = smem + kb * 32768;
      const uint8_t* sb = sa + 16384;
      for (int k = 0; k < BK / 8; ++k) {
        const uint64_t ad = smem_desc_sw128(sa + k * 32, 16, 1024);
        uint64_t bd;
        if (variant == 0) {  // MN-major, SWIZZLE_128B_BASE32B, SBO = 4 rows
          bd = smem_desc_sw128(sb + k * 1024, 4096, 512);
          bd = (bd & ~(7ull << 61)) | (1ull << 61);
        } else if (variant == 1) {  // BASE32B with SBO = 8 rows
          bd = smem_desc_sw128(sb + k * 1024, 4096, 1024);
          bd = (bd & ~(7ull << 61)) | (1ull << 61);
        } else {  // K-major B^T tile: 128 rows (n) x 32 k, like A
          bd = smem_desc_sw128(sb + k * 32, 16, 1024);
        }
        mma_tf32(tmem, ad, bd, idesc, (kb | k) != 0);
      }
    }
    tc_commit(&tfull);
  } else if (warp >= 2) {
    const int q = warp & 3;
    mbar_wait(&tfull, 0);
    tc_fence_after();
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      for (int j = 0; j < 32; ++j) C[(q * 32 + lane) * N + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  // dump all four stages (128 KB)
  for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x)
    dump[i] = reinterpret_cast<float*>(smem)[i];
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

static float encB(int k, int n) { return static_cast<float>((k % 32) * 64 + (n % 64)); }

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  std::vector<float> hA(M * K, 0.f), hB(K * N), hC(M * N), hD(4 * 32768 / 4);
  for (int i = 0; i < M; ++i) hA[i * K + i] = 1.0f;
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) hB[k * N + n] = encB(k, n) + (k / 32) * 4096.0f * 0;
  float *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, hA.size() * 4);
  cudaMalloc(&dB, hB.size() * 4);
  cudaMalloc(&dC, hC.size() * 4);
  cudaMalloc(&dD, hD.size() * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb, tb32, tbt;
  std::vector<float> hBt(N * K);
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) hBt[n * K + k] = hB[k * N + n];
  float* dBt;
  cudaMalloc(&dBt, hBt.size() * 4);
  cudaMemcpy(dBt, hBt.data(), hBt.size() * 4, cudaMemcpyHostToDevice);
  {
    cuuint64_t dims[2] = {K, M}, str[1] = {K * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    printf("encA %d\n", enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[2] = {N, K}, str[1] = {N * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    printf("encB %d\n", enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[2] = {N, K}, str[1] = {N * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    printf("encB32 %d\n", enc(&tb32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[2] = {K, N}, str[1] = {K * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    printf("encBt %d\n", enc(&tbt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dBt, dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  const size_t smem = 1024 + 4 * 32768;
  cudaFuncSetAttribute(dbg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int variant = 0; variant < 3; ++variant) {
    if (only >= 0 && variant != only) continue;
    cudaMemset(dC, 0, hC.size() * 4);
    dbg_kernel<<<1, 192, smem>>>(ta, variant == 2 ? tbt : tb32, dC, dD, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) continue;
    cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    if (variant == 99) {
      // check the TMA swizzled images of stage 0
      int badA = 0, badB = 0;
      const uint8_t* d = reinterpret_cast<const uint8_t*>(hD.data());
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 32; ++k) {
          const int atom = m / 8, r = m % 8, chunk = k / 4;
          const int off = atom * 1024 + r * 128 + ((chunk ^ r) * 16) + (k % 4) * 4;
          float v;
          memcpy(&v, d + off, 4);
          if (v != hA[m * K + k]) ++badA;
        }
      for (int n = 0; n < 128; ++n)
        for (int k = 0; k < 32; ++k) {
          const int box = n / 32, nn = n % 32, atom = k / 8, r = k % 8, chunk = nn / 4;
          const int off = 16384 + box * 4096 + atom * 1024 + r * 128 + ((chunk ^ r) * 16) + (nn % 4) * 4;
          float v;
          memcpy(&v, d + off, 4);
          if (v != hB[k * N + n]) ++badB;
        }
      printf("TMA image mismatches: A %d / 4096, B %d / 4096\n", badA, badB);
    }
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n)
        if (hC[m * N + n] != hB[m * N + n]) ++bad;
    printf("variant %d: C mismatches %d / %d\n", variant, bad, M * N);
    for (int m : {0, 1, 2, 8, 33, 127}) {
      printf(" row %3d:", m);
      for (int n : {0, 1, 2, 3, 4, 31, 32, 64, 127}) {
        const float v = hC[m * N + n];
        printf(" %8.1f", v);
      }
      printf("   want:");
      for (int n : {0, 1, 2, 3, 4, 31, 32, 64, 127}) printf(" %6.0f", hB[m * N + n]);
      printf("\n");
    }
  }
  return 0;
}
