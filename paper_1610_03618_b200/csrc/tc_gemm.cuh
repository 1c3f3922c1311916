// Warp-specialised tcgen05 (kind::tf32) GEMM machinery for sm_100a,
// parameterised by an operand Loader (which TMA boxes fill a pipeline stage)
// and an output sink (where the accumulator tile goes).  Shared by the plain
// GEMM (gemm.cu) and the CHWN implicit-GEMM convolution (conv.cu); the NCHW
// gather convolution (conv.cu) reuses the constants and barriers.
//
//   D[M=128 x N] (TMEM, fp32) += A[128 x BK] (smem, K-major, SW128)
//                               x B[BK x N] (smem, K- or MN-major)
//
// Roles: warp 0 = TMA producer (one thread), warp 1 = MMA issuer (one
// thread), warps 2..5 = epilogue (TMEM lane quarter = warp % 4).
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

// ---------------------------------------------------------------------------
// Persistent tcgen05 GEMM: one CTA per SM walks a static tile schedule.
// Tiles are 128 (M) x 256 (N) -- one UMMA_N = 256 instruction per K-step, so
// each A tile is reused across twice the columns -- and the fp32 accumulator
// is double-buffered in TMEM (2 x 256 of the 512 columns): while the four
// epilogue warps drain tile i, the MMA warp already accumulates tile i+1, and
// the TMA warp streams operands through a kPStages-deep shared-memory ring
// without ever stopping between tiles.
//
// Loader concept (the producer thread calls begin() once per tile, then
// load() for k-blocks 0..kblocks(z)-1 of each segment in order, so loaders can
// decode K incrementally instead of dividing per stage):
//   uint32_t kblocks(uint32_t z) const;      // k-blocks of BK in split z
//   uint32_t segments() const;               // chained operand sets (1 or 3)
//   void prefetch() const;                   // tensor-map prefetch
//   State begin(uint32_t m0, uint32_t n0, uint32_t z) const;
//   void load(State& st, uint32_t seg, uint32_t kb, void* sa, void* sb,
//             uint64_t* bar) const;         // issues TMA, total kPStageBytes
//   static constexpr bool kBMajorMN;         // B operand major-ness
// Out concept:
//   void store32(uint32_t m, uint32_t n0, const float* v) const;  // 32 columns
constexpr int kPBN = 256, kPStages = 4;
constexpr uint32_t kPBBytes = kTcBK * kPBN * 4;            // 32 KB
constexpr uint32_t kPStageBytes = kTcABytes + kPBBytes;    // 48 KB
constexpr size_t kPSmem = 1024 + kPStages * kPStageBytes + 256;

struct PCtl {
  uint64_t full[kPStages];
  uint64_t empty[kPStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_addr;
};

struct TileGrid {
  uint32_t mt, nt, splits;  // tiles along M, tiles along N, K splits
};

template <class Loader, class Out>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_persistent(const __grid_constant__ Loader ld, const __grid_constant__ Out out,
                       TileGrid tg) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  PCtl* ctl = reinterpret_cast<PCtl*>(smem + kPStages * kPStageBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t per_split = tg.mt * tg.nt;
  const uint32_t total = per_split * tg.splits;

  if (warp == 0) {
    if (lane == 0) {
      ld.prefetch();
      for (int s = 0; s < kPStages; ++s) {
        mbar_init(&ctl->full[s], 1);
        mbar_init(&ctl->empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&ctl->tfull[a], 1);
        mbar_init(&ctl->tempty[a], 4);  // one arrive per epilogue warp
      }
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<512>(&ctl->tmem_addr);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_addr;

  auto decode = [&](uint32_t t, uint32_t& m0, uint32_t& n0, uint32_t& z) {
    z = t / per_split;
    const uint32_t r = t - z * per_split;
    const uint32_t nt = r / tg.mt;
    m0 = (r - nt * tg.mt) * kTcBM;
    n0 = nt * kPBN;
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    uint32_t s = 0, phase = 0;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
      uint32_t m0, n0, z;
      decode(t, m0, n0, z);
      auto st = ld.begin(m0, n0, z);
      const uint32_t kbn = ld.kblocks(z), segs = ld.segments();
      for (uint32_t seg = 0; seg < segs; ++seg)
        for (uint32_t kb = 0; kb < kbn; ++kb) {
          mbar_wait(&ctl->empty[s], phase ^ 1);
          uint8_t* sa = smem + s * kPStageBytes;
          mbar_arrive_expect_tx(&ctl->full[s], kPStageBytes);
          ld.load(st, seg, kb, sa, sa + kTcABytes, &ctl->full[s]);
          if (++s == kPStages) {
            s = 0;
            phase ^= 1;
          }
        }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_tf32(kTcBM, kPBN, false, Loader::kBMajorMN);
    uint32_t s = 0, phase = 0, local = 0;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      uint32_t m0, n0, z;
      decode(t, m0, n0, z);
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      mbar_wait(&ctl->tempty[a], aphase ^ 1);  // epilogue drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + a * kPBN;
      const uint32_t steps = ld.kblocks(z) * ld.segments();
      for (uint32_t it = 0; it < steps; ++it) {
        mbar_wait(&ctl->full[s], phase);
        tc_fence_after();
        const uint8_t* sa = smem + s * kPStageBytes;
        const uint8_t* sb = sa + kTcABytes;
#pragma unroll
        for (int k = 0; k < kTcBK / 8; ++k) {
          const uint64_t ad = smem_desc_sw128(sa + k * 32, 16, 1024);
          const uint64_t bd = Loader::kBMajorMN ? smem_desc_sw128(sb + k * 1024, 4096, 512, 1)
                                                : smem_desc_sw128(sb + k * 32, 16, 1024);
          mma_tf32(acc, ad, bd, idesc, (it | k) != 0);
        }
        tc_commit(&ctl->empty[s]);
        if (++s == kPStages) {
          s = 0;
          phase ^= 1;
        }
      }
      tc_commit(&ctl->tfull[a]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    uint32_t local = 0;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      uint32_t m0, n0, z;
      decode(t, m0, n0, z);
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      mbar_wait(&ctl->tfull[a], aphase);
      tc_fence_after();
      const uint32_t m = m0 + q * 32 + lane;
      const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < kPBN; c += 32) {
        float v[32];
        tmem_ld32(base + c, v);
        out.store32(m, n0 + c, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->tempty[a]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace lcnn_tc
