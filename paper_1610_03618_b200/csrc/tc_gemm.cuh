// Generic warp-specialised tcgen05 (kind::tf32) GEMM mainloop for sm_100a,
// parameterised by an operand Loader (which TMA boxes fill a pipeline stage)
// and an output sink (where the accumulator tile goes).  Shared by the plain
// GEMM (gemm.cu) and the implicit-GEMM convolutions (conv.cu).
//
//   D[M=128 x N=128] (TMEM, fp32) += A[128 x BK] (smem, K-major, SW128)
//                                   x B[BK x 128] (smem, K- or MN-major, SW128)
//
// Roles: warp 0 = TMA producer (one thread), warp 1 = MMA issuer (one
// thread), warps 2..5 = epilogue (TMEM lane quarter = warp % 4).
// A stage is BK = 32 fp32 of K: A 16 KB + B 16 KB; kStages deep ring.
// A K-step of the MMA is 8 tf32 (32 bytes): K-major operands advance their
// descriptor start by 32 B inside the 128-B swizzle row (SWIZZLE_128B),
// MN-major operands by 8 rows (1024 B) of the SWIZZLE_128B_BASE32B layout
// that tf32 requires for MN-major (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
// The pipeline can chain several "segments" (sets of operands) into one
// accumulator -- used by the 3xTF32 mode (hi*hi + hi*lo + lo*hi).
#pragma once

#include "tc.cuh"

namespace lcnn_tc {

constexpr int kTcBM = 128, kTcBN = 128, kTcBK = 32, kTcStages = 4;
constexpr uint32_t kTcABytes = kTcBM * kTcBK * 4;  // 16 KB
constexpr uint32_t kTcBBytes = kTcBK * kTcBN * 4;  // 16 KB
constexpr uint32_t kTcStageBytes = kTcABytes + kTcBBytes;
constexpr int kTcThreads = 192;
constexpr size_t kTcSmem = 1024 + kTcStages * kTcStageBytes + 256;

struct TcCtl {
  uint64_t full[kTcStages];
  uint64_t empty[kTcStages];
  uint64_t tmem_full;
  uint32_t tmem_addr;
};

// Loader concept (the producer thread calls begin() once per tile, then
// load() for k-blocks 0..kblocks()-1 of each segment in order, so loaders can
// decode K incrementally instead of dividing per stage):
//   uint32_t kblocks() const;                 // k-blocks of BK per segment
//   uint32_t segments() const;                // chained operand sets (1 or 3)
//   void prefetch() const;                    // tensor-map prefetch
//   State begin(uint32_t m0, uint32_t ntile) const;
//   void load(State& st, uint32_t seg, uint32_t kb, void* sa, void* sb,
//             uint64_t* bar) const;          // issues TMA, total kTcStageBytes
//   static constexpr bool kBMajorMN;          // B operand major-ness
// Out concept:
//   void store32(uint32_t m, uint32_t ntile, uint32_t col, const float* v) const;
template <class Loader, class Out>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const __grid_constant__ Loader ld, const __grid_constant__ Out out) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  TcCtl* ctl = reinterpret_cast<TcCtl*>(smem + kTcStages * kTcStageBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t m0 = blockIdx.y * kTcBM;
  const uint32_t ntile = blockIdx.x;
  const uint32_t kb_per_seg = ld.kblocks();
  const uint32_t total = kb_per_seg * ld.segments();

  if (warp == 0) {
    if (lane == 0) {
      ld.prefetch();
      for (int s = 0; s < kTcStages; ++s) {
        mbar_init(&ctl->full[s], 1);
        mbar_init(&ctl->empty[s], 1);
      }
      mbar_init(&ctl->tmem_full, 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<128>(&ctl->tmem_addr);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_addr;

  if (warp == 0 && lane == 0) {
    auto st = ld.begin(m0, ntile);
    uint32_t seg = 0, kb = 0, s = 0, phase = 0;
    for (uint32_t it = 0; it < total; ++it) {
      mbar_wait(&ctl->empty[s], phase ^ 1);
      uint8_t* sa = smem + s * kTcStageBytes;
      mbar_arrive_expect_tx(&ctl->full[s], kTcStageBytes);
      ld.load(st, seg, kb, sa, sa + kTcABytes, &ctl->full[s]);
      if (++kb == kb_per_seg) {
        kb = 0;
        ++seg;
      }
      if (++s == kTcStages) {
        s = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_tf32(kTcBM, kTcBN, false, Loader::kBMajorMN);
    uint32_t s = 0, phase = 0;
    for (uint32_t it = 0; it < total; ++it) {
      mbar_wait(&ctl->full[s], phase);
      tc_fence_after();
      const uint8_t* sa = smem + s * kTcStageBytes;
      const uint8_t* sb = sa + kTcABytes;
#pragma unroll
      for (int k = 0; k < kTcBK / 8; ++k) {
        const uint64_t ad = smem_desc_sw128(sa + k * 32, 16, 1024);
        // MN-major B: 32-float atoms 4096 B apart along N, 4-row groups 512 B
        // apart along K (BASE32B); one MMA K-step = 8 rows = 1024 B.
        const uint64_t bd = Loader::kBMajorMN ? smem_desc_sw128(sb + k * 1024, 4096, 512, 1)
                                              : smem_desc_sw128(sb + k * 32, 16, 1024);
        mma_tf32(tmem, ad, bd, idesc, (it | k) != 0);
      }
      tc_commit(&ctl->empty[s]);
      if (++s == kTcStages) {
        s = 0;
        phase ^= 1;
      }
    }
    tc_commit(&ctl->tmem_full);
  } else if (warp >= 2) {
    const int q = warp & 3;
    mbar_wait(&ctl->tmem_full, 0);
    tc_fence_after();
    const uint32_t m = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < kTcBN; c += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      out.store32(m, ntile, c, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

}  // namespace lcnn_tc
