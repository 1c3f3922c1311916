// Convolution for the whole-network path (conv.hpp:17-54).
//
// Reference: /root/reference/proj/src/conv.cpp
//   conv_direct_chwn  :102-152  CHWN, image block innermost
//   conv_direct_nchw  :157-196  NCHW, window innermost
//   conv_gemm + im2col:215-332  materialised unroll + blocked GEMM
//   conv_oracle       :53-93    fp64 ground truth
//
// B200 design -- CHWN implicit GEMM on tcgen05 (no im2col in HBM):
//   D[(oh, ow, n)][co] = sum_k X[(oh, ow, n)][k] * Wpack[co][k]
// The GEMM M index (oh, ow, n) is exactly the CHWN output column order and the
// output channels are the N side (UMMA N = C_o up to 256, so 96 / 192
// channel layers waste nothing on a 128-row tile).  A tiles are TMA boxes of
// the 4D input (n, w, h, c) -- the batch is contiguous, so every k-row of a
// tile is 32 images (128 B) of one input pixel: an MN-major operand in the
// SWIZZLE_128B_BASE32B layout tf32 requires.
// Padding is TMA out-of-bounds zero fill (negative / overflowing h, w
// coordinates).  Two K orderings:
//   CI  (C_i % 32 == 0): k = (fh, fw, ci); a k-block is 32 channels of one
//        filter tap: box {32 n, 1 w, 1 h, 32 c}.
//   WIN (F_w <= 16):     k = (fh, ci, fw'); fw padded to FP in {4, 8, 16};
//        a k-block is 32/FP channels x FP taps of one filter row:
//        box {32 n, FP w, 1 h, 32/FP c}; padded taps get zero weights.
// Filters are packed once per call into the matching K-major [co][K] matrix.
// 3xTF32 mode chains hi*hi + hi*lo + lo*hi over split copies of both operands.
//
// The fp32 SIMT kernels serve LCNN_PREC_FP32 (bit-level fp32 products, the
// host API's default for reference-tolerance parity) and every shape the
// tensor-core path does not cover (NCHW, batches that are not a multiple of
// 32, rectangular windows wider than 16).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "../../include/lcnn_cuda.h"
#include "common.cuh"
#include "internal.h"
#include "tc_gemm.cuh"

namespace lcnn_dev {

using namespace lcnn_tc;

enum ConvMode : uint32_t { kModeCI = 0, kModeWIN = 1, kModeNAT = 2, kModeROW = 3, kModeSHARE = 4,
                          kModeTAPS = 5 };

struct ConvGeomTc {
  uint32_t N, Ci, H, W, Co, FH, FW, S, P, Ho, Wo;
  uint32_t mode, FP, CIB, CiP;
  uint32_t KR;  // ROW mode: k-rows per filter row (Ci*FP rounded up to 8; FP = row width)
};

// Wpack[co][k] in the loader's K order, zero for padded (ci, fw) slots.
__global__ void pack_filters_kernel(const float* __restrict__ f, float* __restrict__ hi,
                                    float* __restrict__ lo, ConvGeomTc g, uint32_t K) {
  const uint64_t total = static_cast<uint64_t>(g.Co) * K;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t co = static_cast<uint32_t>(i / K);
    const uint32_t k = static_cast<uint32_t>(i % K);
    uint32_t ci, fh, fw;
    bool valid = true;
    if (g.mode == kModeCI) {
      ci = k % g.Ci;
      const uint32_t tap = k / g.Ci;
      fh = tap / g.FW;
      fw = tap % g.FW;
    } else if (g.mode == kModeTAPS) {  // k = (fh, channel block, fw, 32 channels)
      const uint32_t c = k % 32, q = k / 32;
      fw = q % g.FW;
      const uint32_t t = q / g.FW, cb = t % (g.Ci / 32);
      fh = t / (g.Ci / 32);
      ci = cb * 32 + c;
    } else if (g.mode == kModeROW) {  // k = (fh, ci, fw), each fh row padded to KR
      fh = k / g.KR;
      const uint32_t r = k - fh * g.KR;
      ci = r / g.FW;
      fw = r - ci * g.FW;
      valid = ci < g.Ci;
    } else if (g.mode == kModeNAT) {  // natural (ci, fh, fw) order, K padded
      fw = k % g.FW;
      fh = (k / g.FW) % g.FH;
      ci = k / (g.FW * g.FH);
      valid = ci < g.Ci;
    } else {
      fw = k % g.FP;
      const uint32_t t = k / g.FP;
      ci = t % g.CiP;
      fh = t / g.CiP;
      valid = fw < g.FW && ci < g.Ci;
    }
    float v = 0.0f;
    if (valid) v = f[((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw];
    if (lo) {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
      const float h = __uint_as_float(r);
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v - h));
      hi[i] = h;
      lo[i] = __uint_as_float(r);
    } else {
      hi[i] = v;
    }
  }
}

// TAPS row-pair filter image (C_o <= 64, stride 1): 128 rows x K2, K2 =
// (FH + 1) * Ci * FW in the TAPS order with the filter row replaced by the
// INPUT row offset dr = 0..FH of a two-output-row tile: row r < 64 is
// channel r of output row oh (filter row fh = dr), row r >= 64 channel r - 64
// of output row oh + 1 (fh = dr - 1); out-of-range filter rows and channels
// are zero.
__global__ void pack_filters_taps2_kernel(const float* __restrict__ f, float* __restrict__ out,
                                          ConvGeomTc g, uint32_t K2) {
  const uint64_t total = 128ull * K2;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t row = static_cast<uint32_t>(i / K2), k = static_cast<uint32_t>(i % K2);
    const uint32_t c = k % 32, q = k / 32;
    const uint32_t fw = q % g.FW, t = q / g.FW, cb = t % (g.Ci / 32), dr = t / (g.Ci / 32);
    const uint32_t co = row & 63u, ci = cb * 32 + c;
    const int fh = static_cast<int>(dr) - (row >= 64 ? 1 : 0);
    float v = 0.0f;
    if (co < g.Co && fh >= 0 && fh < static_cast<int>(g.FH))
      v = f[((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw];
    out[i] = v;
  }
}

// The implicit im2col of the CHWN input is the MN-major operand: 4D TMA boxes
// of 32 output columns (32 images of one output pixel) x 32 k-rows.  The
// packed filters [co][K] are the K-major operand: one 2D box of 32 k x (tile
// width) output channels.  kCoOnN picks the orientation:
//   true : A = input (4 boxes = 128 columns), B = filters (N = bn channels)
//   false: A = filters (128 channels),        B = input (8 boxes = 256 columns)
// kPair: the CTA-pair kernel (tc_gemm_pair) -- this CTA's 128 input columns
// and half of the channel tile's filter rows, completing on the leader's
// barrier (channels on N only).
template <bool kCoOnN, bool kPair = false>
struct ChwnConvLoader {
  CUtensorMap x[2];  // input hi / lo          (4D: {N, W, H, Ci}, or grouped 5D)
  CUtensorMap w[2];  // packed filters hi / lo (2D: {K, Co})
  ConvGeomTc g;
  uint32_t ncols;  // Ho*Wo*N
  // grouped (N % 128 == 0): the input view {32 n, W, Ci, N/32, H} -- group
  // stride 128 B -- so ONE 5D box {32, FP, CIB, 4, 1} lands a whole
  // 128-column block (one output pixel, 4 MN-major atoms) instead of four
  // 4D boxes; TMA cost is mostly per box (scripts/tma_bench.cu)
  bool grouped;
  static constexpr bool kAMajorMN = kCoOnN, kBMajorMN = !kCoOnN, kZeroSmem = false;
  static constexpr bool kResidentA = false;
  static constexpr int kSteps = kTcBK / 8;
  static constexpr int kBoxes = kCoOnN ? kTcBM / 32 : kPBN / 32;
  // input image: SWIZZLE_128B_BASE32B, 32-column atoms of 32 k-rows (4 KB);
  // filters: K-major SWIZZLE_128B, 8-row groups of 1 KB
  __device__ uint64_t desc_a(const uint8_t* sa, int k) const {
    return kCoOnN ? smem_desc_sw128(sa + k * 1024, 4096, 512, 1)
                  : smem_desc_sw128(sa + k * 32, 16, 1024);
  }
  __device__ uint64_t desc_b(const uint8_t* sb, int k) const {
    return kCoOnN ? smem_desc_sw128(sb + k * 32, 16, 1024)
                  : smem_desc_sw128(sb + k * 1024, 4096, 512, 1);
  }
  __device__ void prefetch() const {
    tma_prefetch(&x[0]);
    tma_prefetch(&w[0]);
  }
  __device__ uint32_t resident_bytes() const { return 0; }
  __device__ void load_resident(void*, uint64_t*) const {}
  __device__ uint32_t resident_offset(uint32_t) const { return 0; }
  // Per tile fragment: the column boxes' (n0, w origin, h origin) and the
  // first k-block's (fh, fw, channel) decoded once; per k-block the tap /
  // channel-block counters advance incrementally.  Grouped: entry j < kBoxes/4
  // describes 128-column block j and n0 holds its first group index.
  struct State {
    uint32_t co0;
    int32_t n0[kBoxes], y0[kBoxes], z0[kBoxes];
    uint32_t fh, wofs, c0;  // K decode of the next k-block
  };
  __device__ State begin(uint32_t m0, uint32_t n0, uint32_t kfirst) const {
    State st;
    const uint32_t col0 = kCoOnN ? m0 : n0;
    st.co0 = kCoOnN ? n0 : m0;
    const uint32_t span = grouped ? 128 : 32;
#pragma unroll
    for (int j = 0; j < kBoxes; ++j) {
      const uint32_t col = col0 + span * j;
      const uint32_t pos = col / g.N;
      const uint32_t oh = pos / g.Wo, ow = pos - oh * g.Wo;
      const uint32_t nn = col - pos * g.N;
      st.n0[j] = static_cast<int32_t>(grouped ? nn / 32 : nn);
      st.y0[j] = static_cast<int32_t>(ow * g.S) - static_cast<int32_t>(g.P);
      // beyond the last output: an all-out-of-bounds box (zeros)
      st.z0[j] = col >= ncols ? -(1 << 20)
                              : static_cast<int32_t>(oh * g.S) - static_cast<int32_t>(g.P);
    }
    if (g.mode == kModeCI) {
      const uint32_t cpb = g.Ci / 32, r = kfirst / cpb;
      st.c0 = (kfirst - r * cpb) * 32;
      st.fh = r / g.FW;
      st.wofs = r - st.fh * g.FW;
    } else {
      const uint32_t cpb = g.CiP / g.CIB;
      st.fh = kfirst / cpb;
      st.c0 = (kfirst - st.fh * cpb) * g.CIB;
      st.wofs = 0;
    }
    return st;
  }
  __device__ void load(State& st, uint32_t seg, uint32_t k, void* sa, void* sb,
                       uint64_t* bar) const {
    if (k == 0) st.fh = st.wofs = st.c0 = 0;  // a new segment restarts K
    uint8_t* sx = static_cast<uint8_t*>(kCoOnN ? sa : sb);
    const CUtensorMap* xm = &x[seg == 1 ? 1 : 0];
    if constexpr (kPair) {
      static_assert(kCoOnN, "pair mode puts the input columns on M");
      const uint32_t lb = mapa_shared(smem_u32(bar), 0);  // the leader's full barrier
      if (grouped) {
        tma_load_5d_cg2(sx, xm, lb, 0, st.y0[0] + static_cast<int32_t>(st.wofs),
                        static_cast<int32_t>(st.c0), st.n0[0],
                        st.z0[0] + static_cast<int32_t>(st.fh));
      } else {
#pragma unroll
        for (int j = 0; j < kBoxes; ++j)
          tma_load_4d_cg2(sx + j * 4096, xm, lb, st.n0[j], st.y0[j] + static_cast<int32_t>(st.wofs),
                          st.z0[j] + static_cast<int32_t>(st.fh), static_cast<int32_t>(st.c0));
      }
      tma_load_2d_cg2(sb, &w[seg == 2 ? 1 : 0], lb, k * kTcBK, st.co0);
    } else {
      if (grouped) {
#pragma unroll
        for (int j = 0; j < kBoxes / 4; ++j)
          tma_load_5d(sx + j * 16384, xm, bar, 0, st.y0[j] + static_cast<int32_t>(st.wofs),
                      static_cast<int32_t>(st.c0), st.n0[j], st.z0[j] + static_cast<int32_t>(st.fh));
      } else {
#pragma unroll
        for (int j = 0; j < kBoxes; ++j)
          tma_load_4d(sx + j * 4096, xm, bar, st.n0[j], st.y0[j] + static_cast<int32_t>(st.wofs),
                      st.z0[j] + static_cast<int32_t>(st.fh), static_cast<int32_t>(st.c0));
      }
      tma_load_2d(kCoOnN ? sb : sa, &w[seg == 2 ? 1 : 0], bar, k * kTcBK, st.co0);
    }
    // advance: CI mode k = (fh, fw, ci/32); WIN mode k = (fh, ci/CIB)
    if (g.mode == kModeCI) {
      st.c0 += 32;
      if (st.c0 == g.Ci) {
        st.c0 = 0;
        if (++st.wofs == g.FW) {
          st.wofs = 0;
          ++st.fh;
        }
      }
    } else {
      st.c0 += g.CIB;
      if (st.c0 == g.CiP) {
        st.c0 = 0;
        ++st.fh;
      }
    }
  }
};

// ROW mode (small C_i * F_w, e.g. AlexNet conv1: 3 x 11): a pipeline stage
// is one whole filter row, k = (ci, fw) in the order a single box
// {32 n, F_w w, 1 h, C_i c} lays rows down, padded only to the MMA K-step of
// 8 (33 -> 40 rows instead of WIN's 3 -> 4 channels x 11 -> 16 taps = 64).
// Channels are the N side.  The filters are pre-packed in global memory as
// the exact shared-memory image of the B operand per (channel tile, filter
// row) -- the SWIZZLE_NONE K-major core-matrix layout, [k/4][bn][4].
// Resident mode (one channel tile, TF32, image fits next to >= 3 ring
// slots): the whole filter image -- 169 KB for conv1 -- is bulk-copied into
// shared memory ONCE per CTA and every stage streams only the input boxes
// (halving conv1's per-stage operand bytes); otherwise a stage's B is one
// contiguous bulk copy of bn * KR * 4 bytes.  The padding rows of the input
// boxes are never written by TMA; the kernel zeroes shared memory once at
// start (kZeroSmem) and the padded weights are zero.
template <bool kCoOnN>
struct ChwnRowLoader {
  CUtensorMap x[2];         // input hi / lo (4D: {N, W, H, Ci}, box {32, FW, 1, Ci})
  const float* wimg[2];     // filter images hi / lo: [co tile][fh][KR/4][bn][4]
  ConvGeomTc g;
  uint32_t ncols, bn;       // bn: channel rows per filter-image tile (the N or M extent)
  uint32_t res;             // resident filter image bytes (0 = streamed per stage)
  // grouped (N % 128 == 0): 5D view {32 n, W, Ci, N/32, H}, one box
  // {32, FP, Ci, 4, 1} per 128-column block; each group's rows are (ci, w)
  // with w padded to FP so a group is exactly KR = Ci * FP rows (whole
  // 1 KB swizzle atoms); the padded taps have zero weights
  bool grouped;
  // row pairs (channels on M, C_o <= 64, stride 1): columns are (row pair,
  // ow, n), g.FH counts the F_h + 1 input rows of a pair (RowsPairOut)
  bool rows2;
  static constexpr bool kAMajorMN = kCoOnN, kBMajorMN = !kCoOnN, kZeroSmem = true;
  static constexpr bool kResidentA = false;
  static constexpr int kSteps = 0;
  static constexpr int kBoxes = kCoOnN ? kTcBM / 32 : kPBN / 32;  // 32-column input boxes
  // input operand: MN-major SWIZZLE_128B_BASE32B, kBoxes groups of KR rows;
  // filter operand: K-major SWIZZLE_NONE core matrices [k/4][bn][4]
  __device__ uint64_t desc_x(const uint8_t* p, int k) const {
    return smem_desc_sw128(p + k * 1024, g.KR * 128, 512, 1);
  }
  __device__ uint64_t desc_w(const uint8_t* p, int k) const {
    // K-step k = k-chunks 2k, 2k+1; LBO = next k-chunk, SBO = next 8 rows
    return smem_desc_sw128(p + 2 * k * bn * 16, bn * 16, 128, 0);
  }
  __device__ uint64_t desc_a(const uint8_t* sa, int k) const {
    return kCoOnN ? desc_x(sa, k) : desc_w(sa, k);
  }
  __device__ uint64_t desc_b(const uint8_t* sb, int k) const {
    return kCoOnN ? desc_w(sb, k) : desc_x(sb, k);
  }
  __device__ void prefetch() const { tma_prefetch(&x[0]); }
  __device__ uint32_t resident_bytes() const { return res; }
  __device__ void load_resident(void* dst, uint64_t* bar) const {
    const uint32_t row = g.KR * bn * 4;  // one filter row per copy
    for (uint32_t fh = 0; fh < g.FH; ++fh)
      bulk_load(static_cast<uint8_t*>(dst) + fh * row, wimg[0] + fh * g.KR * bn, row, bar);
  }
  __device__ uint32_t resident_offset(uint32_t kb) const { return kb * g.KR * bn * 4; }
  struct State {
    uint32_t wofs, fh;  // filter image offset of this channel tile (floats), filter row
    int32_t n0[kBoxes], y0[kBoxes], z0[kBoxes];
  };
  __device__ State begin(uint32_t m0, uint32_t n0, uint32_t kfirst) const {
    State st;
    const uint32_t col0 = kCoOnN ? m0 : n0, co0 = kCoOnN ? n0 : m0;
    st.wofs = co0 / bn * g.FH * g.KR * bn;
    st.fh = kfirst;
    const uint32_t span = grouped ? 128 : 32;
#pragma unroll
    for (int j = 0; j < kBoxes; ++j) {
      const uint32_t col = col0 + span * j;
      const uint32_t pos = col / g.N;
      const uint32_t ohp = pos / g.Wo, ow = pos - ohp * g.Wo, oh = rows2 ? 2 * ohp : ohp;
      const uint32_t nn = col - pos * g.N;
      st.n0[j] = static_cast<int32_t>(grouped ? nn / 32 : nn);
      st.y0[j] = static_cast<int32_t>(ow * g.S) - static_cast<int32_t>(g.P);
      st.z0[j] = col >= ncols ? -(1 << 20)
                              : static_cast<int32_t>(oh * g.S) - static_cast<int32_t>(g.P);
    }
    return st;
  }
  __device__ void load(State& st, uint32_t seg, uint32_t k, void* sa, void* sb,
                       uint64_t* bar) const {
    if (k == 0) st.fh = 0;
    const CUtensorMap* xm = &x[seg == 1 ? 1 : 0];
    uint8_t* sx = static_cast<uint8_t*>(kCoOnN ? sa : sb);
    if (grouped) {
#pragma unroll
      for (int j = 0; j < kBoxes / 4; ++j)
        tma_load_5d(sx + j * 4 * g.KR * 128, xm, bar, 0, st.y0[j], 0, st.n0[j],
                    st.z0[j] + static_cast<int32_t>(st.fh));
    } else {
#pragma unroll
      for (int j = 0; j < kBoxes; ++j)
        tma_load_4d(sx + j * g.KR * 128, xm, bar, st.n0[j], st.y0[j],
                    st.z0[j] + static_cast<int32_t>(st.fh), 0);
    }
    if (!res)
      bulk_load(kCoOnN ? sb : sa, wimg[seg == 2 ? 1 : 0] + st.wofs + st.fh * g.KR * bn,
                g.KR * bn * 4, bar);
    ++st.fh;
  }
};

// Filter image of ROW mode: img[((t * FH + fh) * KR/4 + q) * bn + r][e] =
// W[co = t*bn + r][ci][fh][fw] with ci*FP + fw = 4q + e (FP = the row width:
// F_w, or its padding in grouped mode; zero when padded).
__global__ void pack_filters_row_kernel(const float* __restrict__ f, float* __restrict__ hi,
                                        float* __restrict__ lo, ConvGeomTc g, uint32_t bn,
                                        uint64_t total) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = static_cast<uint32_t>(i & 3);
    uint64_t rest = i >> 2;
    const uint32_t r = static_cast<uint32_t>(rest % bn);
    rest /= bn;
    const uint32_t q = static_cast<uint32_t>(rest % (g.KR / 4));
    rest /= g.KR / 4;
    const uint32_t fh = static_cast<uint32_t>(rest % g.FH);
    const uint32_t t = static_cast<uint32_t>(rest / g.FH);
    const uint32_t kk = 4 * q + e, co = t * bn + r;
    uint32_t ci, fw;
    if (g.mode == kModeSHARE) {  // k = (fw, ci): channels fastest
      fw = kk / g.Ci;
      ci = kk - fw * g.Ci;
    } else {  // k = (ci, fw)
      ci = kk / g.FP;
      fw = kk - ci * g.FP;
    }
    float v = 0.0f;
    if (co < g.Co && ci < g.Ci && fw < g.FW)
      v = f[((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw];
    if (lo) {
      uint32_t u;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
      const float h = __uint_as_float(u);
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v - h));
      hi[i] = h;
      lo[i] = __uint_as_float(u);
    } else {
      hi[i] = v;
    }
  }
}

// Row-pair ROW image (C_o <= 64, stride 1): img[(dr * KR/4 + q) * 128 + r][e]
// for input row offset dr = 0..FH of a two-output-row tile; row r < 64 is
// channel r of output row oh (filter row fh = dr), r >= 64 channel r - 64 of
// row oh + 1 (fh = dr - 1); zero outside the filter.
__global__ void pack_filters_row2_kernel(const float* __restrict__ f, float* __restrict__ hi,
                                         ConvGeomTc g, uint64_t total) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = static_cast<uint32_t>(i & 3);
    const uint64_t rest = i >> 2;
    const uint32_t r = static_cast<uint32_t>(rest % 128);
    const uint32_t q = static_cast<uint32_t>((rest / 128) % (g.KR / 4));
    const uint32_t dr = static_cast<uint32_t>(rest / 128 / (g.KR / 4));
    const uint32_t kk = 4 * q + e, co = r & 63u;
    const int fh = static_cast<int>(dr) - (r >= 64 ? 1 : 0);
    const uint32_t ci = kk / g.FP, fw = kk - ci * g.FP;
    float v = 0.0f;
    if (co < g.Co && ci < g.Ci && fw < g.FW && fh >= 0 && fh < static_cast<int>(g.FH))
      v = f[((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw];
    hi[i] = v;
  }
}

// Row-pair output (ChwnRowLoader::rows2): accumulator rows 0-63 are output
// row 2p's channels, 64-127 row 2p + 1's; tile columns are (p, ow, n).  A
// 32 x 32 chunk never straddles the halves or a pixel, so it maps to one
// TMA box of the RowsOut view {ncols, C_o}.
// kPairs: chunks staged two at a time with one async-proxy fence (the
// short-K SHARE epilogue's scheme; VGG conv1_1 is store-bound: 424 us with
// stores vs 188 us without, PROFILING probe)
template <bool kPairs, bool kTma = true>
struct RowsPairOutT {
  float* c;
  uint64_t ldc;       // real columns Ho * Wo * N
  uint32_t M, span, ho;  // C_o, Wo * N, Ho
  CUtensorMap y;
  static constexpr bool kTmaStore = kTma, kTmaTransposed = false, kTmaPairs = kPairs;
  __device__ __forceinline__ bool remap(uint32_t& m, uint32_t& n) const {
    const uint32_t pr = n / span, oh = 2 * pr + (m >= 64 ? 1u : 0u);
    m &= 63u;
    n = oh * span + (n - pr * span);
    return oh < ho;
  }
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    if (!remap(m0, n0) || m0 >= M) return;
    if (add)
      tma_add_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
    else
      tma_store_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    if (!remap(m, n0)) return;  // warp-uniform (one pixel, one half)
    warp_store_rows32(m < M ? c + m * ldc + n0 : nullptr, v, add);
  }
};

// Row-pair output with quad-chunk stores (OutTmaQuads): a tile's 128
// consecutive columns of one output row (one pixel x 128 images at N = 128)
// go out as one box per 32 channels, 512 B per channel, through the 3D view
// yq {32, ncols / 32, C_o}; split tiles (stream-K fragments) and tiles whose
// columns are not 128-aligned use the 2D chunk path of RowsPairOutT.
//
// Blocked output (nimg != 0, LCNN_CONV_OUT_HWCN32): the activation is
// [N/32][H][W][C][32], so a (pixel, 32-image group) holds its C channels' 128-B
// lines contiguously and a quad box is four 4 KB runs.  y / yq are then 4D
// views {32 i, N/32 g, H*W pixel, C} (boxes {32, 1, 1, 32} / {32, 4, 1, 32}).
struct RowsQuadOut : RowsPairOutT<false> {
  CUtensorMap yq;
  uint32_t nimg = 0, hw = 0;  // blocked: images N, pixels Ho * Wo
  static constexpr bool kTmaQuads = true;
  __device__ __forceinline__ void tma_quad(const void* box, uint32_t m0, uint32_t n0) const {
    if (!remap(m0, n0) || m0 >= M) return;
    if (nimg)
      tma_store_4d(&yq, box, 0, static_cast<int32_t>(n0 % nimg / 32),
                   static_cast<int32_t>(n0 / nimg), static_cast<int32_t>(m0));
    else
      tma_store_3d(&yq, box, 0, static_cast<int32_t>(n0 / 32), static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    if (!nimg) return RowsPairOutT<false>::tma_chunk(box, m0, n0, add);
    if (!remap(m0, n0) || m0 >= M) return;
    const int32_t g = static_cast<int32_t>(n0 % nimg / 32), px = static_cast<int32_t>(n0 / nimg);
    if (add)
      tma_add_4d(&y, box, 0, g, px, static_cast<int32_t>(m0));
    else
      tma_store_4d(&y, box, 0, g, px, static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    if (!nimg) return RowsPairOutT<false>::store32(m, n0, v, add);
    if (!remap(m, n0)) return;  // warp-uniform
    const uint64_t line = (uint64_t{n0 % nimg / 32} * hw + n0 / nimg) * M + m;
    warp_store_rows32(m < M ? c + line * 32 : nullptr, v, add);
  }
};

struct RowsOut {  // accumulator rows = channels: C[co][col], ldc = ncols (a multiple of 32)
  float* c;
  uint64_t ldc;
  uint32_t M, N;
  uint32_t keep_l2 = 0;  // TMA stores with an L2 evict_last hint (the next layer reads them)
  // TMA-store epilogue: 2D view {N cols, M rows} (pitch ldc), box {32, 32},
  // SWIZZLE_128B; out-of-range rows / columns of a box are clipped
  CUtensorMap y;
  static constexpr bool kTmaStore = true, kTmaTransposed = false;
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    if (n0 >= N || m0 >= M) return;
    if (add)
      tma_add_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
    else if (keep_l2)
      tma_store_2d_keep(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
    else
      tma_store_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    if (n0 >= N) return;  // warp-uniform
    if (n0 + 32 <= N) {
      warp_store_rows32(m < M ? c + m * ldc + n0 : nullptr, v, add);
    } else if (m < M) {
      store_row32(c + m * ldc + n0, n0, N, v, add);
    }
  }
};

// Accumulator row m = output column (oh, ow, n), columns = output channels:
// out[co][col] (CHWN).  For each channel the 32 lanes of a warp hold 32
// consecutive columns, so every store instruction is one coalesced 128 B line.
template <bool kTma>
struct ColsOutT {
  float* c;
  uint32_t ncols, co;
  uint32_t keep_l2 = 0;  // TMA stores with an L2 evict_last hint (profiling knob LCNN_KEEP_L2)
  // TMA-store epilogue (kTma): the RowsOut view {ncols, C_o}; a chunk is
  // 32 accumulator rows (columns of C) x 32 channels, staged transposed
  CUtensorMap y;
  static constexpr bool kTmaStore = kTma, kTmaTransposed = true;
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    if (m0 >= ncols || n0 >= co) return;
    if (add)
      tma_add_2d(&y, box, static_cast<int32_t>(m0), static_cast<int32_t>(n0));
    else if (keep_l2)
      tma_store_2d_keep(&y, box, static_cast<int32_t>(m0), static_cast<int32_t>(n0));
    else
      tma_store_2d(&y, box, static_cast<int32_t>(m0), static_cast<int32_t>(n0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    if (m >= ncols) return;
    float* p = c + static_cast<uint64_t>(n0) * ncols + m;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (n0 + j >= co) break;
      if (add)
        atomicAdd(p + static_cast<uint64_t>(j) * ncols, v[j]);
      else
        lcnn_tc::st_out(p + static_cast<uint64_t>(j) * ncols, v[j]);
    }
  }
};
using ColsOut = ColsOutT<true>;
using ColsOutPlain = ColsOutT<false>;

// SHARE mode (small C_i * F_w and C_o <= 128, e.g. AlexNet conv1: 3 x 11,
// stride 4).  A tile is 8 consecutive output pixels of one output row x one
// 32-image group, and ONE TMA box per filter row serves all 8 pixels: the
// input view {32 n, C_i, W, N/32, H} lands the box {32, C_i, BW = S*7 + F_w,
// 1, 1} as rows ordered (w, c), c fastest, so pixel p's receptive-field row
// is the same K sequence k = fw * C_i + c shifted by p * S * C_i rows.  The 8
// MN-major 32-column atoms of the UMMA B operand (N = 256) therefore overlap
// in shared memory at a uniform pitch of S * C_i rows (the descriptor LBO):
// TMA and tcgen05 both swizzle by shared-memory address (verified on B200,
// scripts/swz_test.cu), so an atom may start at any 128-byte row.  The input
// stream per 256 output columns is one box of BW * C_i rows (117 for conv1)
// instead of ROW mode's eight 48-row atoms.  The filters are the A operand
// (channels on M), K-major SWIZZLE_NONE core matrices [fh][KR/4][bn][4] with
// bn = C_o rounded to 8.  The box is latency-bound (one
// 128-B run per row), so the ring depth matters more than the filter bytes:
// the filter row travels with each stage (one contiguous bulk copy, 15 KB for
// conv1) and 7 slots fit, rather than a resident 169 KB image with 3 slots
// (scripts/tma_bench.cu: 38 -> 75 B/clk/SM from 3 to 8 slots).  Rows
// bn..127 of the M = 128 MMA read the next chunk's rows (finite), producing
// accumulator rows no one stores.  K padding rows
// (C_i*F_w .. KR) carry zero weights; the slot rows past the box are never
// written and stay zero.
constexpr uint32_t kSharePix = 8;  // output pixels per tile (8 x 32 columns = UMMA N 256)

struct ChwnShareLoader {
  CUtensorMap x;
  const float* wimg;
  ConvGeomTc g;
  uint32_t bn;      // filter image rows (C_o rounded up to 8)
  uint32_t owb;     // 8-pixel blocks per output row
  uint32_t groups;  // N / 32
  uint32_t res;     // resident filter image bytes
  static constexpr bool kZeroSmem = true;
  static constexpr bool kResidentA = true;
  static constexpr int kSteps = 0;
  __device__ uint64_t desc_a(const uint8_t* sa, int k) const {
    return smem_desc_sw128(sa + 2 * k * bn * 16, bn * 16, 128, 0);
  }
  __device__ uint64_t desc_b(const uint8_t* sb, int k) const {
    return smem_desc_sw128(sb + k * 1024, g.S * g.Ci * 128, 512, 1);
  }
  __device__ void prefetch() const { tma_prefetch(&x); }
  __device__ uint32_t resident_bytes() const { return res; }
  __device__ void load_resident(void* dst, uint64_t* bar) const {
    const uint32_t row = g.KR * bn * 4;  // one filter row per copy
    for (uint32_t fh = 0; fh < g.FH; ++fh)
      bulk_load(static_cast<uint8_t*>(dst) + fh * row, wimg + fh * g.KR * bn, row, bar);
  }
  __device__ uint32_t resident_offset(uint32_t kb) const { return kb * g.KR * bn * 4; }
  struct State {
    int32_t y0, z0, grp;
  };
  __device__ State begin(uint32_t, uint32_t n0, uint32_t) const {
    const uint32_t t = n0 / (kSharePix * 32);
    const uint32_t grp = t % groups, r = t / groups;
    const uint32_t ob = r % owb, oh = r / owb;
    return State{static_cast<int32_t>(ob * kSharePix * g.S) - static_cast<int32_t>(g.P),
                 static_cast<int32_t>(oh * g.S) - static_cast<int32_t>(g.P),
                 static_cast<int32_t>(grp)};
  }
  __device__ void load(State& st, uint32_t, uint32_t k, void* sa, void* sb, uint64_t* bar) const {
    tma_load_5d(sb, &x, bar, 0, 0, st.y0, st.grp, st.z0 + static_cast<int32_t>(k));
    if (!res) bulk_load(sa, wimg + k * g.KR * bn, g.KR * bn * 4, bar);
  }
};

// Accumulator rows = channels, 32-column chunk j = pixel j of the tile's 8
// (its 32 images): out[co][oh][ow][32 grp .. 32 grp + 31], one 128-B line.
struct ShareOut {
  float* c;
  uint64_t plane;  // Ho * Wo * N
  uint32_t co, n, wo, owb, groups;
  // TMA-store epilogue: view {32 n, N/32, Wo, Ho, Co} of the output, box
  // {32, 1, 1, 1, 32} = one 32-channel x 32-image chunk, SWIZZLE_128B
  CUtensorMap y;
  FastDiv fd_groups, fd_owb;  // set by the launcher (TMA-store epilogue)
  uint32_t evict_first = 0;   // TMA stores with an L2 evict_first hint (TAPS, LCNN_TAPS_L2 bit 2)
  static constexpr bool kTmaStore = true, kTmaTransposed = false, kTmaPairs = true;
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    const uint32_t t = n0 / (kSharePix * 32), p = n0 % (kSharePix * 32) / 32;
    uint32_t r, grp, oh, ob;
    fd_groups.divmod(t, r, grp);
    fd_owb.divmod(r, oh, ob);
    const uint32_t ow = ob * kSharePix + p;
    if (ow >= wo || m0 >= co) return;  // (rows past C_o inside the box are clipped)
    if (add)
      tma_add_5d(&y, box, 0, static_cast<int32_t>(grp), static_cast<int32_t>(ow),
                 static_cast<int32_t>(oh), static_cast<int32_t>(m0));
    else if (evict_first)
      tma_store_5d_hint(&y, box, 0, static_cast<int32_t>(grp), static_cast<int32_t>(ow),
                        static_cast<int32_t>(oh), static_cast<int32_t>(m0), l2_policy_evict_first());
    else
      tma_store_5d(&y, box, 0, static_cast<int32_t>(grp), static_cast<int32_t>(ow),
                   static_cast<int32_t>(oh), static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    const uint32_t t = n0 / (kSharePix * 32), p = n0 % (kSharePix * 32) / 32;
    const uint32_t grp = t % groups, r = t / groups;
    const uint32_t ob = r % owb, oh = r / owb, ow = ob * kSharePix + p;
    if (ow >= wo) return;  // warp-uniform
    warp_store_rows32(
        m < co ? c + m * plane + (static_cast<uint64_t>(oh) * wo + ow) * n + grp * 32 : nullptr, v,
        add);
  }
};

// ---- SHARE convolution with the max pooling that follows it fused in ------
// (AlexNet conv1 -> pool1: conv 96 f11 s4 -> 55x55, max 3x3/s2 -> 27x27.)
// The conv output never reaches HBM: a CTA owns one POOLING STRIP -- one
// 32-image group x PC pool columns x a segment of pool rows -- and walks its
// conv rows top to bottom, one tile per row.  A tile is the TPX = 2*(PC-1) +
// PWIN conv pixels the strip's PC windows cover (7 for 3x3/s2: pixels
// 6j..6j+6 serve pool columns 3j..3j+2), UMMA N = 32 * TPX, with the SHARE
// operand layout (one input box per filter row, overlapping MN atoms).  The
// epilogue warps keep the open pool row (PC x 32 images per channel lane) in
// registers across tiles: per window u, h = max of the row's PWIN pixels,
// then pool = max(running, h).  With the reference's compare-select
// (max_tap: NaN never replaces, ties keep the earlier tap) the row-then-column
// order is bit-identical to its (y, x) tap order (the first maximal tap of
// the earlier row wins either way), and each conv value is the same
// K-ordered tensor-core sum as in the unfused SHARE kernel, so the fused
// layer equals conv -> pool_layout bit for bit.  Cost: the strip segments
// recompute one conv row at each boundary and 7 conv pixels serve 6 columns
// (~1.2x the MMA work of the unfused conv), against the unfused output
// stream (149 MB for conv1) and the pooling pass that re-reads it.
// Pooling stride 2 with windows 2 or 3 (one open pool row at a time).
constexpr uint32_t kPoolStride = 2;
template <int PWIN>
struct SharePoolDims {
  static constexpr uint32_t PC = (kSharePix - PWIN) / kPoolStride + 1;  // pool columns per tile
  static constexpr uint32_t TPX = kPoolStride * (PC - 1) + PWIN;         // conv pixels per tile
};

struct ChwnSharePoolLoader : ChwnShareLoader {
  uint32_t units, strips, segs, hp, tpx, pc;
  FastDiv fd_units, fd_groups;
  __device__ State begin(uint32_t, uint32_t n0, uint32_t) const {
    uint32_t k, unit, j, grp;
    fd_units.divmod(n0 / (tpx * 32), k, unit);
    const uint32_t sg = unit / strips, strip = unit - sg * strips;
    fd_groups.divmod(strip, j, grp);
    const uint32_t ph0 = sg * hp / segs, ph1 = (sg + 1) * hp / segs;
    const uint32_t rows = 2 * (ph1 - ph0) + (tpx - kPoolStride * (pc - 1)) - 2;
    const uint32_t oh = kPoolStride * ph0 + (k < rows ? k : rows - 1);  // past the segment: reload its last row
    return State{static_cast<int32_t>(j * pc * kPoolStride * g.S) - static_cast<int32_t>(g.P),
                 static_cast<int32_t>(oh * g.S) - static_cast<int32_t>(g.P),
                 static_cast<int32_t>(grp)};
  }
};

// kDirect: each lane stores its channel's 32 pooled images (one 128-B line)
// straight from registers -- no staging boxes, so the input ring gets their
// 32 KB (one more slot); otherwise a swizzled box per warp and a TMA store.
template <int PWIN, bool kDirect>
struct SharePoolOut {
  static constexpr bool kStateful = true;
  static constexpr uint32_t PC = SharePoolDims<PWIN>::PC;
  // pooled output view {32 n, N/32, Wp, Hp, Co}, box {32, 1, 1, 1, 32}: one
  // 32-channel x 32-image chunk of one pool pixel, SWIZZLE_128B
  CUtensorMap y;
  float* out;  // CHWN [co][hp][wp][n] (kDirect)
  uint32_t n;
  uint32_t co, wp, hp, strips, segs;
  FastDiv fd_units, fd_groups;
  struct Acc {
    float cur[PC][32];  // the open pool row: running max per window, 32 images
  };
  __device__ __forceinline__ void tile(Acc& acc, uint32_t t, uint32_t taddr, uint8_t* stg,
                                       uint32_t& epi_buf, int q, int lane) const {
    uint32_t k, unit, j, grp;
    fd_units.divmod(t, k, unit);
    const uint32_t sg = unit / strips, strip = unit - sg * strips;
    fd_groups.divmod(strip, j, grp);
    const uint32_t ph0 = sg * hp / segs, ph1 = (sg + 1) * hp / segs;
    const uint32_t rows = 2 * (ph1 - ph0) + PWIN - 2;
    const uint32_t m0 = static_cast<uint32_t>(q) * 32;
    if (k >= rows || m0 >= co) return;  // warp-uniform: padding row of the segment / channels
    const uint32_t d = k & 1, i = k >> 1;
    // the pool row this conv row completes (d == 0: the row above's window
    // for 3-wide windows; d == 1: its own for 2-wide ones)
    const bool closes = PWIN == 3 ? (d == 0 && i >= 1) : (d == 1);
    const uint32_t ph = ph0 + (PWIN == 3 ? i - 1 : i);
#pragma unroll
    for (uint32_t u = 0; u < PC; ++u) {
      const uint32_t pw = j * PC + u;
      if (pw >= wp) break;  // warp-uniform
      float h[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) h[e] = -INFINITY;
#pragma unroll
      for (int p = 0; p < PWIN; ++p) {
        float v[32];
        tmem_ld32(taddr + (kPoolStride * u + p) * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) h[e] = max_tap(h[e], v[e]);
      }
      if (closes && kDirect) {
        if (m0 + lane < co) {
          float4* dst = reinterpret_cast<float4*>(
              out + ((static_cast<uint64_t>(m0 + lane) * hp + ph) * wp + pw) * n + grp * 32);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            dst[c] = make_float4(max_tap(acc.cur[u][4 * c], h[4 * c]),
                                 max_tap(acc.cur[u][4 * c + 1], h[4 * c + 1]),
                                 max_tap(acc.cur[u][4 * c + 2], h[4 * c + 2]),
                                 max_tap(acc.cur[u][4 * c + 3], h[4 * c + 3]));
        }
      } else if (closes) {
        uint8_t* box = stg + (epi_buf & 1) * 4096;
        ++epi_buf;
        if (lane == 0) bulk_wait_read_n<1>();  // this box's previous store has read it
        __syncwarp();
        float4* row = reinterpret_cast<float4*>(box + lane * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          row[c ^ (lane & 7)] = make_float4(
              max_tap(acc.cur[u][4 * c], h[4 * c]), max_tap(acc.cur[u][4 * c + 1], h[4 * c + 1]),
              max_tap(acc.cur[u][4 * c + 2], h[4 * c + 2]),
              max_tap(acc.cur[u][4 * c + 3], h[4 * c + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_5d(&y, box, 0, static_cast<int32_t>(grp), static_cast<int32_t>(pw),
                       static_cast<int32_t>(ph), static_cast<int32_t>(m0));
          bulk_commit();
        }
      }
      if (d == 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) acc.cur[u][e] = h[e];  // opens pool row ph0 + i
      } else if (PWIN == 3) {
#pragma unroll
        for (int e = 0; e < 32; ++e) acc.cur[u][e] = max_tap(acc.cur[u][e], h[e]);
      }
    }
  }
};

// ---- TAPS mode: tap-sharing input boxes for CI convolutions ----------------
// A tile is 8 consecutive output pixels of one output row x one 32-image
// group (UMMA N = 256, channels on M, the ShareOut mapping).  K runs (filter
// row fh, 32-channel block cb, tap fw, channel): one input box {32 n, 32 c,
// BW = 7*S + F_w w} per (fh, cb) -- rows ordered (w, c), c fastest -- serves
// all F_w taps of that filter row, tap fw's 8 MN atoms starting fw*4 KB into
// the box at a pitch of S*4 KB (address-swizzled atoms, scripts/swz_test.cu).
// Versus one box per (tap, channel block) that is F_w times fewer input
// bytes per MMA (3x for 3x3 layers, 5x for 5x5).  The filter slices ride a
// separate, deeper ring (16 KB per tap), so an input box stays resident while
// its F_w taps are consumed.
struct TapsCtl {
  uint64_t ifull[4], iempty[4];
  uint64_t ffull[8], fempty[8];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem_addr;
};

struct TapsParams {
  CUtensorMap x;  // input view {32 n, Ci, W, N/32, H}, box {32, 32, BW, 1, 1}
  CUtensorMap w;  // packed filters [Co][K], box {32 k, 128 co}
  Sched sc;       // mt = channel tiles, nt = Ho * OWB * G, iters = FH * CB (stream-K ready)
  ShareOut out;
  uint32_t FW, S, P, CB, OWB, G;
  uint32_t ni, nf, islot, ibox;  // input / filter ring slots, input slot and box bytes
  uint32_t ctl_off;
  // ROW PAIRS (C_o <= 64, stride 1): a tile is two output rows; accumulator
  // rows 0-63 are output row oh, 64-127 row oh + 1, the K loop runs over the
  // FH + 1 input rows they share (pack_filters_taps2_kernel), so the 128-row
  // MMA carries no padding rows and each input box serves both output rows
  uint32_t rows2, Ho;
  // TMA-store epilogue (ShareOut boxes staged at epi_off, two 4 KB boxes per
  // epilogue warp) instead of per-lane stores
  uint32_t tma, epi_off;
  uint32_t in_keep;  // input boxes with an L2 evict_last hint (LCNN_TAPS_L2 bit 1)
  // 2x2 / stride-2 max pooling fused into the row-pair epilogue: a row pair
  // is exactly one pooled row, a 8-pixel block four pooled pixels, so every
  // window lies inside one tile; the conv output never reaches HBM.  The
  // pooled CHWN [co][hp][wp][n] goes to pool_out (whole tiles only, no
  // stream-K); the two rows meet through the epi_off staging (2 x 16 KB)
  float* pool_out;
  uint32_t pool, hp, wp;
  uint32_t FH;  // filter rows (tc_conv_taps_acc2_kernel)
};

__global__ void __launch_bounds__(kTcThreads, 1) tc_conv_taps_kernel(const __grid_constant__ TapsParams prm) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ibase = smem;
  uint8_t* fbase = smem + prm.ni * prm.islot;
  TapsCtl* ctl = reinterpret_cast<TapsCtl*>(smem + prm.ctl_off);
  const Sched& sc = prm.sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&prm.x);
      tma_prefetch(&prm.w);
      for (uint32_t i = 0; i < prm.ni; ++i) {
        mbar_init(&ctl->ifull[i], 1);
        mbar_init(&ctl->iempty[i], 1);
      }
      for (uint32_t i = 0; i < prm.nf; ++i) {
        mbar_init(&ctl->ffull[i], 1);
        mbar_init(&ctl->fempty[i], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&ctl->tfull[a], 1);
        mbar_init(&ctl->tempty[a], 4);
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
  LCNN_PDL_ENTRY();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: input boxes and filter slices ----------------
    uint32_t is = 0, iph = 0, fs = 0, fph = 0;
    // PROFILING probe bit 8: filter slices loaded for the first tile only
    // (later tiles reuse whatever the ring holds): the cost of re-streaming them
    bool reload = true;
    for_each_work(sc, [&](uint32_t t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t mi = t % sc.mt, ni = t / sc.mt;
      const uint32_t g = ni % prm.G, r = ni / prm.G, ob = r % prm.OWB,
                     oh = (r / prm.OWB) << prm.rows2;  // rows2: first row of the pair
      const int32_t y0 = static_cast<int32_t>(ob * kSharePix * prm.S) - static_cast<int32_t>(prm.P);
      const int32_t z0 = static_cast<int32_t>(oh * prm.S) - static_cast<int32_t>(prm.P);
      const int32_t co0 = static_cast<int32_t>(mi * kTcBM);
      for (uint32_t it = kbeg; it < kend; ++it) {
        const uint32_t fh = it / prm.CB, cb = it - fh * prm.CB;
        mbar_wait(&ctl->iempty[is], iph ^ 1);
        mbar_arrive_expect_tx(&ctl->ifull[is], prm.ibox);
        if (prm.in_keep)
          tma_load_5d_hint(ibase + is * prm.islot, &prm.x, &ctl->ifull[is], 0,
                           static_cast<int32_t>(cb * 32), y0, static_cast<int32_t>(g),
                           z0 + static_cast<int32_t>(fh), l2_policy_evict_last());
        else
          tma_load_5d(ibase + is * prm.islot, &prm.x, &ctl->ifull[is], 0,
                      static_cast<int32_t>(cb * 32), y0, static_cast<int32_t>(g),
                      z0 + static_cast<int32_t>(fh));
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          mbar_wait(&ctl->fempty[fs], fph ^ 1);
          if (reload) {
            mbar_arrive_expect_tx(&ctl->ffull[fs], kTcABytes);
            tma_load_2d(fbase + fs * kTcABytes, &prm.w, &ctl->ffull[fs],
                        static_cast<int32_t>((it * prm.FW + fw) * kTcBK), co0);
          } else {
            mbar_arrive(&ctl->ffull[fs]);
          }
          if (++fs == prm.nf) {
            fs = 0;
            fph ^= 1;
          }
        }
      }
      if (sc.probe & 8) reload = false;
    });
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform, one elected lane) ----------------
    const bool mma_on = !(sc.probe & 1);
    const uint32_t lbo = prm.S * 4096;
    uint32_t is = 0, iph = 0, fs = 0, fph = 0, local = 0;
    for_each_work(sc, [&](uint32_t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      mbar_wait(&ctl->tempty[a], aphase ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + a * kPBN;
      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->ifull[is], iph);
        tc_fence_after();
        const uint8_t* xb = ibase + is * prm.islot;
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          mbar_wait(&ctl->ffull[fs], fph);
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(fbase + fs * kTcABytes, 16, 1024);
          const uint64_t db = smem_desc_sw128(xb + fw * 4096, lbo, 512, 1);
          if (elect_one()) {
            if (mma_on) {
#pragma unroll
              for (int k = 0; k < kTcBK / 8; ++k)
                mma_tf32(acc, da + 2 * k, db + 64 * k, sc.idesc,
                         (it != kbeg || fw != 0 || k != 0) ? 1u : 0u);
            }
            tc_commit(&ctl->fempty[fs]);
          }
          __syncwarp();
          if (++fs == prm.nf) {
            fs = 0;
            fph ^= 1;
          }
        }
        if (elect_one()) tc_commit(&ctl->iempty[is]);
        __syncwarp();
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
      }
      if (elect_one()) tc_commit(&ctl->tfull[a]);
      __syncwarp();
    });
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    uint32_t local = 0, epi_buf = 0, pool_buf = 0;
    bool zwait = sc.zsync != nullptr;  // in-kernel stream-K zeroing (Sched::zsync)
    if (zwait) zero_region_arrive(sc);
    for_each_work(sc, [&](uint32_t t, uint32_t, uint32_t, bool split) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      const uint32_t mi = t % sc.mt;
      uint32_t ni = t / sc.mt;
      mbar_wait(&ctl->tfull[a], aphase);
      tc_fence_after();
      if (zwait && t >= sc.ztile) {
        zero_region_wait(sc.zsync, lane);
        zwait = false;
      }
      uint32_t m = mi * kTcBM + q * 32 + lane;
      bool live = true;
      if (prm.rows2) {  // warps 2-3 (lanes 64-127) hold output row oh + 1
        const uint32_t og = prm.OWB * prm.G, pr = ni / og, rest = ni - pr * og;
        const uint32_t oh = 2 * pr + (q >> 1);
        live = oh < prm.Ho;  // warp-uniform
        ni = oh * og + rest;
        m = (q & 1) * 32 + lane;
      }
      const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
      if (prm.pool) {
        // ni was remapped above; the pooled row is the row pair's index
        const uint32_t og = prm.OWB * prm.G, ph = ni / og / 2, rest = ni % og;
        const uint32_t ob = rest / prm.G, grp = rest - ob * prm.G;
        float* stg = reinterpret_cast<float*>(smem + prm.epi_off);
        // warp-uniform and the same for the four epilogue warps (one tile)
        for (uint32_t u = 0; u < kSharePix / 2 && ph < prm.hp; ++u) {
          const uint32_t pw = ob * (kSharePix / 2) + u;
          if (pw >= prm.wp) break;
          float v0[32], v1[32];
          tmem_ld32(base + 2 * u * 32, v0);
          tmem_ld32(base + (2 * u + 1) * 32, v1);
          float4* row = reinterpret_cast<float4*>(stg + ((pool_buf & 1) * 4 + q) * 1024 + lane * 32);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              h[e] = max_tap(max_tap(-INFINITY, v0[4 * c + e]), v1[4 * c + e]);
            row[c ^ (lane & 7)] = make_float4(h[0], h[1], h[2], h[3]);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          // warp q stores channels 16q .. 16q + 15: lanes 8 apart cover one
          // channel's 32 images (128 B), the pooled max of rows oh and oh + 1
          const float4* st4 = reinterpret_cast<const float4*>(stg + (pool_buf & 1) * 4096);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t c = q * 16 + k * 4 + (lane >> 3), j = lane & 7;
            if (c >= prm.out.co) break;
            const uint32_t off = (c & 31) * 8 + (j ^ (c & 7));
            const float4 top = st4[(c >> 5) * 256 + off], bot = st4[(2 + (c >> 5)) * 256 + off];
            float4* dst = reinterpret_cast<float4*>(
                prm.pool_out + ((static_cast<uint64_t>(c) * prm.hp + ph) * prm.wp + pw) * prm.out.n +
                grp * 32);
            dst[j] = max_tap(top, bot);
          }
          ++pool_buf;
        }
      } else if (prm.tma) {
        if (live)
          epilogue_tile(prm.out, sc, smem + prm.epi_off + q * 2 * 4096, base, m, ni * kPBN, split,
                        epi_buf, lane);
      } else {
#pragma unroll 1
        for (uint32_t c = 0; c < kPBN && live; c += 32) {
          float v[32];
          tmem_ld32(base + c, v);
          if (!(sc.probe & 2)) prm.out.store32(m, ni * kPBN + c, v, split);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->tempty[a]);
    });
    if (prm.tma && lane == 0) bulk_wait_read_n<0>();  // staged boxes read before exit
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  } else if (threadIdx.x == 64 && sc.zsync) {
    zero_region_depart(sc.zsync);
  }
}

// ---- TAPS with two accumulators: row pairs for C_o > 64 -------------------
// A tile is two output rows (oh, oh + 1) x 8 pixels x one 32-image group x a
// 128-channel tile, one 256-column TMEM accumulator per row.  K walks the
// F_h + 1 input rows the pair shares: input row r's box feeds accumulator 0
// with filter row r (r < F_h) and accumulator 1 with filter row r - 1
// (r >= 1), so each input box serves both rows -- (F_h + 1) / 2 boxes per
// output row instead of F_h -- with the usual TAPS filter image and the same
// MMA count.  The 512 columns hold no second buffer; instead each accumulator
// has its own full / empty barrier pair: accumulator 0 is finished one input
// row before accumulator 1, and the next tile needs accumulator 1 only from
// its second input row on, so each drain overlaps MMAs of the other.  Stride
// 1, whole tiles (no stream-K).  pool: the 2 x 2 / stride-2 max pool of the
// two rows, horizontal max per accumulator (row oh's staged in shared memory,
// 16 KB per epilogue warp), pooled rows stored with the coalesced 32-row
// store; the conv output never reaches HBM.
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_conv_taps_acc2_kernel(const __grid_constant__ TapsParams prm) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ibase = smem;
  uint8_t* fbase = smem + prm.ni * prm.islot;
  TapsCtl* ctl = reinterpret_cast<TapsCtl*>(smem + prm.ctl_off);
  const Sched& sc = prm.sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&prm.x);
      tma_prefetch(&prm.w);
      for (uint32_t i = 0; i < prm.ni; ++i) {
        mbar_init(&ctl->ifull[i], 1);
        mbar_init(&ctl->iempty[i], 1);
      }
      for (uint32_t i = 0; i < prm.nf; ++i) {
        mbar_init(&ctl->ffull[i], 1);
        mbar_init(&ctl->fempty[i], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&ctl->tfull[a], 1);
        mbar_init(&ctl->tempty[a], 4);
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
  LCNN_PDL_ENTRY();
  const uint32_t FH = prm.FH;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    uint32_t is = 0, iph = 0, fs = 0, fph = 0;
    auto filter = [&](uint32_t fit, uint32_t fw, int32_t co0) {
      mbar_wait(&ctl->fempty[fs], fph ^ 1);
      mbar_arrive_expect_tx(&ctl->ffull[fs], kTcABytes);
      tma_load_2d(fbase + fs * kTcABytes, &prm.w, &ctl->ffull[fs],
                  static_cast<int32_t>((fit * prm.FW + fw) * kTcBK), co0);
      if (++fs == prm.nf) {
        fs = 0;
        fph ^= 1;
      }
    };
    for_each_work(sc, [&](uint32_t t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t mi = t % sc.mt, ni = t / sc.mt;
      const uint32_t g = ni % prm.G, r = ni / prm.G, ob = r % prm.OWB, oh = 2 * (r / prm.OWB);
      const int32_t y0 = static_cast<int32_t>(ob * kSharePix) - static_cast<int32_t>(prm.P);
      const int32_t z0 = static_cast<int32_t>(oh) - static_cast<int32_t>(prm.P);
      const int32_t co0 = static_cast<int32_t>(mi * kTcBM);
      for (uint32_t it = kbeg; it < kend; ++it) {
        const uint32_t rr = it / prm.CB, cb = it - rr * prm.CB;
        mbar_wait(&ctl->iempty[is], iph ^ 1);
        mbar_arrive_expect_tx(&ctl->ifull[is], prm.ibox);
        tma_load_5d(ibase + is * prm.islot, &prm.x, &ctl->ifull[is], 0,
                    static_cast<int32_t>(cb * 32), y0, static_cast<int32_t>(g),
                    z0 + static_cast<int32_t>(rr));
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          if (rr < FH) filter(rr * prm.CB + cb, fw, co0);
          if (rr >= 1) filter((rr - 1) * prm.CB + cb, fw, co0);
        }
      }
    });
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t lbo = 4096;  // stride 1
    uint32_t is = 0, iph = 0, fs = 0, fph = 0, local = 0;
    for_each_work(sc, [&](uint32_t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t ph = local & 1;
      ++local;
      for (uint32_t it = kbeg; it < kend; ++it) {
        const uint32_t rr = it / prm.CB, cb = it - rr * prm.CB;
        if (cb == 0 && rr <= 1) {  // first MMA into accumulator rr: its drain is done
          mbar_wait(&ctl->tempty[rr], ph ^ 1);
          tc_fence_after();
        }
        mbar_wait(&ctl->ifull[is], iph);
        tc_fence_after();
        const uint8_t* xb = ibase + is * prm.islot;
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          const uint64_t db = smem_desc_sw128(xb + fw * 4096, lbo, 512, 1);
#pragma unroll
          for (uint32_t acc = 0; acc < 2; ++acc) {
            if (acc == 0 ? rr >= FH : rr == 0) continue;
            mbar_wait(&ctl->ffull[fs], fph);
            tc_fence_after();
            const uint64_t da = smem_desc_sw128(fbase + fs * kTcABytes, 16, 1024);
            const bool first = cb == 0 && fw == 0 && rr == acc;
            if (elect_one()) {
              if (!(sc.probe & 1)) {
#pragma unroll
                for (int k = 0; k < kTcBK / 8; ++k)
                  mma_tf32(tmem + acc * kPBN, da + 2 * k, db + 64 * k, sc.idesc,
                           (first && k == 0) ? 0u : 1u);
              }
              tc_commit(&ctl->fempty[fs]);
            }
            __syncwarp();
            if (++fs == prm.nf) {
              fs = 0;
              fph ^= 1;
            }
          }
        }
        if (elect_one()) {
          tc_commit(&ctl->iempty[is]);
          if (cb == prm.CB - 1 && rr == FH - 1) tc_commit(&ctl->tfull[0]);
          if (cb == prm.CB - 1 && rr == FH) tc_commit(&ctl->tfull[1]);
        }
        __syncwarp();
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
      }
    });
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    uint32_t local = 0;
    float* stg = reinterpret_cast<float*>(smem + prm.epi_off) + q * 4096;  // pool: [u][lane][32]
    for_each_work(sc, [&](uint32_t t, uint32_t, uint32_t, bool) {
      const uint32_t ph = local & 1;
      ++local;
      const uint32_t mi = t % sc.mt, ni = t / sc.mt;
      const uint32_t og = prm.OWB * prm.G, pr = ni / og, rest = ni - pr * og;
      const uint32_t m = mi * kTcBM + q * 32 + lane;
      const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
      if (!prm.pool) {
#pragma unroll 1
        for (uint32_t acc = 0; acc < 2; ++acc) {
          mbar_wait(&ctl->tfull[acc], ph);
          tc_fence_after();
          const uint32_t oh = 2 * pr + acc;
          if (oh < prm.Ho) {
            const uint32_t n0 = (oh * og + rest) * kPBN;
#pragma unroll 1
            for (uint32_t c = 0; c < kPBN; c += 32) {
              float v[32];
              tmem_ld32(tmem + acc * kPBN + lanes + c, v);
              if (!(sc.probe & 2)) prm.out.store32(m, n0 + c, v, false);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctl->tempty[acc]);
        }
      } else {
        const uint32_t ob = rest / prm.G, grp = rest - ob * prm.G;
#pragma unroll 1
        for (uint32_t acc = 0; acc < 2; ++acc) {
          mbar_wait(&ctl->tfull[acc], ph);
          tc_fence_after();
#pragma unroll 1
          for (uint32_t u = 0; u < kSharePix / 2; ++u) {
            float v0[32], v1[32];
            tmem_ld32(tmem + acc * kPBN + lanes + 2 * u * 32, v0);
            tmem_ld32(tmem + acc * kPBN + lanes + (2 * u + 1) * 32, v1);
            float4* row = reinterpret_cast<float4*>(stg + (u * 32 + lane) * 32);
            if (acc == 0) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                float h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  h[e] = max_tap(max_tap(-INFINITY, v0[4 * c + e]), v1[4 * c + e]);
                row[c ^ (lane & 7)] = make_float4(h[0], h[1], h[2], h[3]);
              }
            } else {
              const uint32_t pw = ob * (kSharePix / 2) + u;
              float o[32];
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float4 top = row[c ^ (lane & 7)];
                const float tv[4] = {top.x, top.y, top.z, top.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  o[4 * c + e] =
                      max_tap(tv[e], max_tap(max_tap(-INFINITY, v0[4 * c + e]), v1[4 * c + e]));
              }
              if (pr < prm.hp && pw < prm.wp && !(sc.probe & 2))  // warp-uniform
                warp_store_rows32(m < prm.out.co ? prm.pool_out +
                                                       ((static_cast<uint64_t>(m) * prm.hp + pr) *
                                                            prm.wp + pw) * prm.out.n + grp * 32
                                                 : nullptr,
                                  o, false);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctl->tempty[acc]);
        }
      }
    });
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---- TAPS-N: tap-sharing boxes with channels on N, on a CTA pair ---------
// The TAPS idea for the L2-resident CI layers (AlexNet conv2-5), oriented
// like the pair kernel: the input is the MN-major A operand and the filters
// the K-major B operand, N = a C_o tile (<= 256, no padding of 192 / 384).
// A CTA's 128 accumulator rows are 4 consecutive output pixels of one output
// row x its 32-image group; the two CTAs of a pair take the two 32-image
// groups of a 64-image block (UMMA M = 256).  K runs (fh, 32-channel block,
// fw, c), the TAPS pack order: one input box {32 n, 32 c, BW = 3*S + F_w w}
// per (fh, block) -- rows (w, c), c fastest -- serves all F_w taps, tap fw's
// 4 MN atoms starting fw * 4 KB into the box at a pitch of S * 4 KB; each
// CTA streams HALF of the tap's filter slice (cta_group::2).  Per CTA and
// (fh, block) that is BW*4 KB + F_w * (C_o tile / 2) * 128 B for 4*F_w MMAs:
// conv2 92 KB per 20 MMAs where the pair CI kernel moves 140 KB.
// Epilogue: warp q holds pixel q's 32 images x the C_o tile; each 32-channel
// chunk is staged transposed (box rows = channels, 128 B of images) and TMA-
// stored into the CHWN output (the ShareOut view), add-reduced for stream-K
// fragments.
struct TapsNCtl {
  uint64_t ifull[4], iempty[4];
  uint64_t ffull[8], fempty[8];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem_addr;
};

struct TapsNParams {
  CUtensorMap x;  // input view {32 n, Ci, W, N/32, H}, box {32, 32, BW, 1, 1}
  CUtensorMap w;  // packed filters [Co][K] (TAPS order), box {32 k, bw/2 co}
  CUtensorMap y;  // output view {32 n, N/32, Wo, Ho, Co}, box {32, 1, 1, 1, 32}
  Sched sc;       // mt = C_o tiles, nt = Ho * OWB * G2, iters = FH * CB
  uint32_t FW, S, P, CB, OWB, G2, Wo, bw;
  uint32_t ni, nf, islot, ibox, fslot;  // ring slots, slot / box bytes (per CTA)
  uint32_t epi_off, ctl_off;
};

constexpr uint32_t kTapsNPix = 4;  // output pixels per CTA tile (4 x 32 images = M 128)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    tc_conv_tapsn_pair_kernel(const __grid_constant__ TapsNParams prm) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ibase = smem;
  uint8_t* fbase = smem + prm.ni * prm.islot;
  TapsNCtl* ctl = reinterpret_cast<TapsNCtl*>(smem + prm.ctl_off);
  const Sched& sc = prm.sc;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&prm.x);
      tma_prefetch(&prm.w);
      for (uint32_t i = 0; i < prm.ni; ++i) {
        mbar_init(&ctl->ifull[i], 1);
        mbar_init(&ctl->iempty[i], 1);
      }
      for (uint32_t i = 0; i < prm.nf; ++i) {
        mbar_init(&ctl->ffull[i], 1);
        mbar_init(&ctl->fempty[i], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&ctl->tfull[a], 1);
        mbar_init(&ctl->tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
      }
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc_cg2<512>(&ctl->tmem_addr);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_addr;
  LCNN_PDL_ENTRY();
  const uint32_t half = prm.bw / 2;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs; completion on the leader) ----------------
    const uint32_t lead_ifull = mapa_shared(smem_u32(&ctl->ifull[0]), 0);
    const uint32_t lead_ffull = mapa_shared(smem_u32(&ctl->ffull[0]), 0);
    uint32_t is = 0, iph = 0, fs = 0, fph = 0;
    for_each_work(sc, pair, npairs, [&](uint32_t t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t mi = t % sc.mt, ni = t / sc.mt;
      const uint32_t g2 = ni % prm.G2, r = ni / prm.G2, ob = r % prm.OWB, oh = r / prm.OWB;
      const int32_t x0 = static_cast<int32_t>(ob * kTapsNPix * prm.S) - static_cast<int32_t>(prm.P);
      const int32_t z0 = static_cast<int32_t>(oh * prm.S) - static_cast<int32_t>(prm.P);
      const int32_t grp = static_cast<int32_t>(2 * g2 + rank);
      const int32_t co0 = static_cast<int32_t>(mi * prm.bw + rank * half);
      for (uint32_t it = kbeg; it < kend; ++it) {
        const uint32_t fh = it / prm.CB, cb = it - fh * prm.CB;
        mbar_wait(&ctl->iempty[is], iph ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&ctl->ifull[is], 2 * prm.ibox);
        tma_load_5d_cg2(ibase + is * prm.islot, &prm.x, lead_ifull + is * 8, 0,
                        static_cast<int32_t>(cb * 32), x0, grp, z0 + static_cast<int32_t>(fh));
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          mbar_wait(&ctl->fempty[fs], fph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&ctl->ffull[fs], 2 * prm.fslot);
          tma_load_2d_cg2(fbase + fs * prm.fslot, &prm.w, lead_ffull + fs * 8,
                          static_cast<int32_t>((it * prm.FW + fw) * kTcBK), co0);
          if (++fs == prm.nf) {
            fs = 0;
            fph ^= 1;
          }
        }
      }
    });
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader, M = 256) ----------------
    const bool mma_on = !(sc.probe & 1);
    const uint32_t lbo = prm.S * 4096;
    uint32_t is = 0, iph = 0, fs = 0, fph = 0, local = 0;
    for_each_work(sc, pair, npairs, [&](uint32_t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      mbar_wait(&ctl->tempty[a], aphase ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + a * kPBN;
      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->ifull[is], iph);
        tc_fence_after();
        const uint8_t* xb = ibase + is * prm.islot;
        for (uint32_t fw = 0; fw < prm.FW; ++fw) {
          mbar_wait(&ctl->ffull[fs], fph);
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(xb + fw * 4096, lbo, 512, 1);
          const uint64_t db = smem_desc_sw128(fbase + fs * prm.fslot, 16, 1024);
          if (elect_one()) {
            if (mma_on) {
#pragma unroll
              for (int k = 0; k < kTcBK / 8; ++k)
                mma_tf32_cg2(acc, da + 64 * k, db + 2 * k, sc.idesc,
                             (it != kbeg || fw != 0 || k != 0) ? 1u : 0u);
            }
            tc_commit_cg2(&ctl->fempty[fs], 3);
          }
          __syncwarp();
          if (++fs == prm.nf) {
            fs = 0;
            fph ^= 1;
          }
        }
        if (elect_one()) tc_commit_cg2(&ctl->iempty[is], 3);
        __syncwarp();
        if (++is == prm.ni) {
          is = 0;
          iph ^= 1;
        }
      }
      if (elect_one()) tc_commit_cg2(&ctl->tfull[a], 3);
      __syncwarp();
    });
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs: own TMEM half) ----------------
    const int q = warp & 3;  // TMEM lane quarter = output pixel q of the tile
    const uint32_t leader_tempty = mapa_shared(smem_u32(&ctl->tempty[0]), 0);
    uint8_t* box = smem + prm.epi_off + q * 4096;
    const uint32_t col = ((static_cast<uint32_t>(lane) >> 2) << 4) | ((lane & 3) << 2);
    uint32_t local = 0;
    bool zwait = sc.zsync != nullptr;  // in-kernel stream-K zeroing (Sched::zsync)
    if (zwait) zero_region_arrive(sc);
    for_each_work(sc, pair, npairs, [&](uint32_t t, uint32_t, uint32_t, bool split) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      const uint32_t mi = t % sc.mt, ni = t / sc.mt;
      const uint32_t g2 = ni % prm.G2, r = ni / prm.G2, ob = r % prm.OWB, oh = r / prm.OWB;
      const uint32_t ow = ob * kTapsNPix + q;
      mbar_wait(&ctl->tfull[a], aphase);
      tc_fence_after();
      if (zwait && t >= sc.ztile) {
        zero_region_wait(sc.zsync, lane);
        zwait = false;
      }
      const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (uint32_t c = 0; c < prm.bw; c += 32) {
        float v[32];
        tmem_ld32(base + c, v);
        if (lane == 0) bulk_wait_read_n<0>();  // the box's previous store has read it
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          *reinterpret_cast<float*>(box + j * 128 + (col ^ ((j & 7) << 4))) = v[j];
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && ow < prm.Wo && !(sc.probe & 2)) {
          const int32_t cz = static_cast<int32_t>(mi * prm.bw + c);
          if (split)
            tma_add_5d(&prm.y, box, 0, static_cast<int32_t>(2 * g2 + rank),
                       static_cast<int32_t>(ow), static_cast<int32_t>(oh), cz);
          else
            tma_store_5d(&prm.y, box, 0, static_cast<int32_t>(2 * g2 + rank),
                         static_cast<int32_t>(ow), static_cast<int32_t>(oh), cz);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + a * 8);
    });
    if (lane == 0) bulk_wait_read_n<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem);
  } else if (threadIdx.x == 64 && sc.zsync) {
    zero_region_depart(sc.zsync);
  }
}

// ---- NCHW implicit GEMM on tcgen05 --------------------------------------
//   D[co][(n, p)] = sum_k W[co][k] * X[k][(n, p)],  k = (ci, fh, fw),
//   p = oh*Wo + ow.  NCHW rows of odd width cannot be TMA tensors (16-byte
//   global stride rule), so the B tile is gathered: 128 producer threads each
//   own one output column, load its 32 K-values of the stage (consecutive
//   lanes = consecutive ow, so stride-1 convolutions read coalesced rows;
//   padding is a bounds check), and write them as 128-bit chunks into a
//   K-major SWIZZLE_128B image (each 8-lane phase hits 8 distinct swizzled
//   16-byte slots: conflict-free), then fence the async proxy and arrive on
//   the stage barrier.  Filters come by TMA (natural K order, zero-padded).
//   Warps 0-3: B gather, warp 4: A TMA, warp 5: MMA, warps 6-9: epilogue.
constexpr int kNchwThreads = 320;

struct NchwConvParams {
  CUtensorMap a;  // packed filters (2D: {K, Co}, box {32, 128})
  const float* x;
  float* y;
  uint32_t Ci, H, W, Co, FH, FW, S, Pad, Ho, Wo, P;
  uint32_t K, kb, ncols;  // true K, k-blocks of 32, N * Ho * Wo
};

__global__ void __launch_bounds__(kNchwThreads, 1)
    tc_conv_nchw_kernel(const __grid_constant__ NchwConvParams prm) {
  LCNN_PDL_ENTRY();
  extern __shared__ uint8_t raw_smem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) &
                                             ~uintptr_t(1023));
  TcCtl* ctl = reinterpret_cast<TcCtl*>(smem + kTcStages * kTcStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t m0 = blockIdx.y * kTcBM;
  const uint32_t ntile = blockIdx.x;
  if (warp == 4) {
    if (lane == 0) {
      tma_prefetch(&prm.a);
      for (int s = 0; s < kTcStages; ++s) {
        mbar_init(&ctl->full[s], 129);  // 128 gather threads + the A TMA arrive
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

  if (warp < 4) {
    // ---------------- B gather producers ----------------
    const uint32_t c = threadIdx.x;  // column of the tile == row of the K-major image
    const uint32_t j = ntile * kTcBN + c;
    const bool valid = j < prm.ncols;
    const uint32_t n = valid ? j / prm.P : 0;
    const uint32_t pp = valid ? j - n * prm.P : 0;
    const uint32_t oh = pp / prm.Wo, ow = pp - oh * prm.Wo;
    const int32_t ih0 = static_cast<int32_t>(oh * prm.S) - static_cast<int32_t>(prm.Pad);
    const int32_t iw0 = static_cast<int32_t>(ow * prm.S) - static_cast<int32_t>(prm.Pad);
    const float* img = prm.x + static_cast<uint64_t>(n) * prm.Ci * prm.H * prm.W;
    const uint32_t r8 = c & 7;
    const uint32_t row_off = (c >> 3) * 1024 + r8 * 128;
    uint32_t ci = 0, fh = 0, fw = 0;  // decode of the next k
    uint32_t s = 0, phase = 0;
    for (uint32_t kb = 0; kb < prm.kb; ++kb) {
      mbar_wait(&ctl->empty[s], phase ^ 1);
      float v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int32_t ih = ih0 + static_cast<int32_t>(fh);
        const int32_t iw = iw0 + static_cast<int32_t>(fw);
        const bool in = valid && ci < prm.Ci && ih >= 0 && ih < static_cast<int32_t>(prm.H) &&
                        iw >= 0 && iw < static_cast<int32_t>(prm.W);
        v[q] = in ? __ldg(img + (static_cast<uint64_t>(ci) * prm.H + ih) * prm.W + iw) : 0.0f;
        if (++fw == prm.FW) {
          fw = 0;
          if (++fh == prm.FH) {
            fh = 0;
            ++ci;
          }
        }
      }
      uint8_t* sb = smem + s * kTcStageBytes + kTcABytes + row_off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(sb + ((q ^ r8) << 4)) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&ctl->full[s]);
      if (++s == kTcStages) {
        s = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 4 && lane == 0) {
    // ---------------- A (filters) TMA producer ----------------
    uint32_t s = 0, phase = 0;
    for (uint32_t kb = 0; kb < prm.kb; ++kb) {
      mbar_wait(&ctl->empty[s], phase ^ 1);
      mbar_arrive_expect_tx(&ctl->full[s], kTcABytes);
      tma_load_2d(smem + s * kTcStageBytes, &prm.a, &ctl->full[s], kb * kTcBK, m0);
      if (++s == kTcStages) {
        s = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 5 && lane == 0) {
    // ---------------- MMA issuer (both operands K-major SW128) ----------------
    constexpr uint32_t idesc = idesc_tf32(kTcBM, kTcBN, false, false);
    uint32_t s = 0, phase = 0;
    for (uint32_t kb = 0; kb < prm.kb; ++kb) {
      mbar_wait(&ctl->full[s], phase);
      tc_fence_after();
      const uint8_t* sa = smem + s * kTcStageBytes;
      const uint8_t* sb = sa + kTcABytes;
#pragma unroll
      for (int k = 0; k < kTcBK / 8; ++k)
        mma_tf32(tmem, smem_desc_sw128(sa + k * 32, 16, 1024), smem_desc_sw128(sb + k * 32, 16, 1024),
                 idesc, (kb | k) != 0);
      tc_commit(&ctl->empty[s]);
      if (++s == kTcStages) {
        s = 0;
        phase ^= 1;
      }
    }
    tc_commit(&ctl->tmem_full);
  } else if (warp >= 6) {
    // ---------------- epilogue: out[n][co][p] ----------------
    const int q = warp & 3;
    mbar_wait(&ctl->tmem_full, 0);
    tc_fence_after();
    const uint32_t co = m0 + q * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < kTcBN; cc += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + cc, v);
      if (co >= prm.Co) continue;
      uint32_t j = ntile * kTcBN + cc;
      if (j >= prm.ncols) continue;
      uint32_t n = j / prm.P, pp = j - n * prm.P;
      float* dst = prm.y + (static_cast<uint64_t>(n) * prm.Co + co) * prm.P + pp;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if (j + t < prm.ncols) *dst = v[t];
        ++dst;
        if (++pp == prm.P) {  // next image: jump to its row of channel co
          pp = 0;
          ++n;
          dst = prm.y + (static_cast<uint64_t>(n) * prm.Co + co) * prm.P;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// ---- fp32 SIMT direct convolution (any shape, CHWN or NCHW) --------------
struct ConvGeomSimt {
  uint32_t N, Ci, H, W, Co, FH, FW, S, P, Ho, Wo;
};

__global__ void __launch_bounds__(256)
    conv_chwn_simt_kernel(const float* __restrict__ x, const float* __restrict__ f,
                          float* __restrict__ y, ConvGeomSimt g) {
  LCNN_PDL_ENTRY();
  const uint64_t total = static_cast<uint64_t>(g.Co) * g.Ho * g.Wo * g.N;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t n = static_cast<uint32_t>(i % g.N);
    uint64_t t = i / g.N;
    const uint32_t ow = static_cast<uint32_t>(t % g.Wo);
    t /= g.Wo;
    const uint32_t oh = static_cast<uint32_t>(t % g.Ho);
    const uint32_t co = static_cast<uint32_t>(t / g.Ho);
    double total = 0.0;  // conv.cpp:121-139: fp32 window sums, fp64 total
    for (uint32_t ci = 0; ci < g.Ci; ++ci) {
      float acc = 0.0f;
      for (uint32_t fh = 0; fh < g.FH; ++fh) {
        const int32_t ih = static_cast<int32_t>(oh * g.S + fh) - static_cast<int32_t>(g.P);
        if (ih < 0 || ih >= static_cast<int32_t>(g.H)) continue;
        for (uint32_t fw = 0; fw < g.FW; ++fw) {
          const int32_t iw = static_cast<int32_t>(ow * g.S + fw) - static_cast<int32_t>(g.P);
          if (iw < 0 || iw >= static_cast<int32_t>(g.W)) continue;
          acc = fmaf(__ldg(x + ((static_cast<uint64_t>(ci) * g.H + ih) * g.W + iw) * g.N + n),
                     __ldg(f + ((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw),
                     acc);
        }
      }
      total += acc;
    }
    y[i] = static_cast<float>(total);
  }
}

__global__ void __launch_bounds__(256)
    conv_nchw_simt_kernel(const float* __restrict__ x, const float* __restrict__ f,
                          float* __restrict__ y, ConvGeomSimt g) {
  LCNN_PDL_ENTRY();
  const uint64_t total = static_cast<uint64_t>(g.N) * g.Co * g.Ho * g.Wo;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t ow = static_cast<uint32_t>(i % g.Wo);
    uint64_t t = i / g.Wo;
    const uint32_t oh = static_cast<uint32_t>(t % g.Ho);
    t /= g.Ho;
    const uint32_t co = static_cast<uint32_t>(t % g.Co);
    const uint32_t n = static_cast<uint32_t>(t / g.Co);
    double total = 0.0;  // conv.cpp:175-189: fp32 window sums, fp64 total
    for (uint32_t ci = 0; ci < g.Ci; ++ci) {
      float acc = 0.0f;
      const float* plane = x + (static_cast<uint64_t>(n) * g.Ci + ci) * g.H * g.W;
      for (uint32_t fh = 0; fh < g.FH; ++fh) {
        const int32_t ih = static_cast<int32_t>(oh * g.S + fh) - static_cast<int32_t>(g.P);
        if (ih < 0 || ih >= static_cast<int32_t>(g.H)) continue;
        for (uint32_t fw = 0; fw < g.FW; ++fw) {
          const int32_t iw = static_cast<int32_t>(ow * g.S + fw) - static_cast<int32_t>(g.P);
          if (iw < 0 || iw >= static_cast<int32_t>(g.W)) continue;
          acc = fmaf(__ldg(plane + static_cast<uint64_t>(ih) * g.W + iw),
                     __ldg(f + ((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw),
                     acc);
        }
      }
      total += acc;
    }
    y[i] = static_cast<float>(total);
  }
}

// fp64 ground truth (conv.cpp:53-93): any input layout via strides, NCHW out.
__global__ void conv_oracle_kernel(const float* __restrict__ x, const float* __restrict__ f,
                                   float* __restrict__ y, ConvGeomSimt g, uint64_t sn, uint64_t sc,
                                   uint64_t sh, uint64_t sw) {
  const uint64_t total = static_cast<uint64_t>(g.N) * g.Co * g.Ho * g.Wo;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t ow = static_cast<uint32_t>(i % g.Wo);
    uint64_t t = i / g.Wo;
    const uint32_t oh = static_cast<uint32_t>(t % g.Ho);
    t /= g.Ho;
    const uint32_t co = static_cast<uint32_t>(t % g.Co);
    const uint32_t n = static_cast<uint32_t>(t / g.Co);
    double acc = 0.0;
    for (uint32_t ci = 0; ci < g.Ci; ++ci)
      for (uint32_t fh = 0; fh < g.FH; ++fh) {
        const int32_t ih = static_cast<int32_t>(oh * g.S + fh) - static_cast<int32_t>(g.P);
        if (ih < 0 || ih >= static_cast<int32_t>(g.H)) continue;
        for (uint32_t fw = 0; fw < g.FW; ++fw) {
          const int32_t iw = static_cast<int32_t>(ow * g.S + fw) - static_cast<int32_t>(g.P);
          if (iw < 0 || iw >= static_cast<int32_t>(g.W)) continue;
          acc += static_cast<double>(x[n * sn + ci * sc + ih * sh + iw * sw]) *
                 static_cast<double>(f[((static_cast<uint64_t>(co) * g.Ci + ci) * g.FH + fh) * g.FW + fw]);
        }
      }
    y[i] = static_cast<float>(acc);
  }
}

// Receptive-field unroll of NCHW input (conv.cpp:215-250): rows (ci, fh, fw),
// columns (n, oh, ow); padded taps are zero.
__global__ void im2col_kernel(const float* __restrict__ x, float* __restrict__ m, ConvGeomSimt g) {
  const uint64_t cols = static_cast<uint64_t>(g.N) * g.Ho * g.Wo;
  const uint64_t total = static_cast<uint64_t>(g.Ci) * g.FH * g.FW * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t col = i % cols, row = i / cols;
    const uint32_t ow = static_cast<uint32_t>(col % g.Wo);
    const uint64_t t = col / g.Wo;
    const uint32_t oh = static_cast<uint32_t>(t % g.Ho);
    const uint32_t n = static_cast<uint32_t>(t / g.Ho);
    const uint32_t fw = static_cast<uint32_t>(row % g.FW);
    const uint32_t fh = static_cast<uint32_t>((row / g.FW) % g.FH);
    const uint32_t ci = static_cast<uint32_t>(row / (static_cast<uint64_t>(g.FW) * g.FH));
    const int32_t ih = static_cast<int32_t>(oh * g.S + fh) - static_cast<int32_t>(g.P);
    const int32_t iw = static_cast<int32_t>(ow * g.S + fw) - static_cast<int32_t>(g.P);
    float v = 0.0f;
    if (ih >= 0 && ih < static_cast<int32_t>(g.H) && iw >= 0 && iw < static_cast<int32_t>(g.W))
      v = x[((static_cast<uint64_t>(n) * g.Ci + ci) * g.H + ih) * g.W + iw];
    m[i] = v;
  }
}

}  // namespace lcnn_dev

namespace lcnn_impl {

cudaError_t launch_conv_oracle(const ConvArgs& a, uint64_t sn, uint64_t sc, uint64_t sh,
                               uint64_t sw, cudaStream_t s) {
  lcnn_dev::ConvGeomSimt g{a.n, a.ci, a.h, a.w, a.co, a.fh, a.fw, a.stride, a.pad, a.ho, a.wo};
  lcnn_dev::conv_oracle_kernel<<<148 * 16, 256, 0, s>>>(a.src, a.filters, a.dst, g, sn, sc, sh, sw);
  return cudaGetLastError();
}

cudaError_t launch_im2col(const ConvArgs& a, cudaStream_t s) {
  lcnn_dev::ConvGeomSimt g{a.n, a.ci, a.h, a.w, a.co, a.fh, a.fw, a.stride, a.pad, a.ho, a.wo};
  lcnn_dev::im2col_kernel<<<148 * 16, 256, 0, s>>>(a.src, a.dst, g);
  return cudaGetLastError();
}

using namespace lcnn_dev;

bool make_tmap_2d(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer,
                  uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer, bool mn_major);
// swizzle: 0 = SWIZZLE_128B, 1 = SWIZZLE_128B_ATOM_32B, 2 = none
bool make_tmap(CUtensorMap* m, const float* base, uint32_t rank, const uint64_t* dims,
               const uint64_t* pitches_bytes, const uint32_t* box, const uint32_t* estrides,
               int swizzle);
cudaError_t launch_split_hilo(const float* x, float* hi, float* lo, uint64_t count,
                              cudaStream_t s);
inline bool make_cols_out_map(CUtensorMap* m, const ColsOut& o) {
  const uint64_t dims[2] = {o.ncols, o.co};
  const uint64_t pitch[1] = {static_cast<uint64_t>(o.ncols) * 4};
  const uint32_t box[2] = {32, 32};
  return make_tmap(m, o.c, 2, dims, pitch, box, nullptr, 0);
}
inline bool make_rows_out_map(CUtensorMap* m, const RowsOut& o) {
  const uint64_t dims[2] = {o.N, o.M};
  const uint64_t pitch[1] = {o.ldc * 4};
  const uint32_t box[2] = {32, 32};
  return make_tmap(m, o.c, 2, dims, pitch, box, nullptr, 0);
}


namespace {

// The CTA-pair conv outputs are TMA-stored with an L2 evict_last hint, so
// the next layer finds them in L2: measured on B200 (two boxes, alternating
// runs), AlexNet conv2 -> pool2 20.7 -> 18.7 us, forward +0.7 / +1.2 %
// (profiles/r02_keep_l2_ab.jsonl).  The same hint on the single-CTA RowsOut
// (conv3-5) measured neutral.  Profiling knob LCNN_KEEP_L2: 0 off, 1 the
// CTA-pair outputs (default), 2 also RowsOut.
int keep_l2_knob() {
  static const int k = [] {
    const char* e = std::getenv("LCNN_KEEP_L2");
    return e ? std::atoi(e) : 1;
  }();
  return k;
}

// Output-channel tile width when channels are the N side: one or two tiles of
// <= 256, rounded to 32 (no padding of C_o = 96 / 192 to a 128-row tile).
uint32_t co_tile_n(uint32_t co) {
  const uint32_t nco = (co + kPBN - 1) / kPBN;
  return ((co + nco - 1) / nco + 31) / 32 * 32;
}

// Measured on B200 (scripts/mma_bench.cu, scripts/tma_bench.cu): one
// tcgen05.mma.kind::tf32 with M = 128, K = 8 occupies the tensor pipe for
// max(~96, N/2) cycles (N = 256: 128 cycles = 1.1 PFLOP/s per chip; N <= 192:
// a ~96-cycle floor, so narrow MMAs waste issue slots), and a TMA box costs
// ~80 cycles of fixed overhead plus ~0.9 cycle per 128-byte row it moves.  A
// pipeline stage takes the longer of the two.
double stage_cycles(uint32_t ksteps, uint32_t bn, uint32_t boxes, uint32_t rows) {
  const double per = bn / 2.0 > 96.0 ? bn / 2.0 : 96.0;
  const double mma = per * ksteps, tma = 80.0 * boxes + 0.9 * rows;
  return mma > tma ? mma : tma;
}

// Orientation by the cost model: channels on N (tiles of 128 columns x
// co_tile_n channels, kTcBM/32 input boxes) or channels on M (128-channel
// tiles x 256 columns, kPBN/32 input boxes) -- the cheaper whole-layer
// estimate wins, ties go to channels on N (fewer boxes).  krows: k-rows per
// stage; in_rows: 128-byte rows of one 32-column input box; w_rows: 128-byte
// rows of one 128-row filter slice of a stage.
bool choose_co_on_n(uint32_t co, uint64_t ncols, uint32_t krows, uint32_t in_rows,
                    uint32_t w_rows_per_128, bool grouped) {
  const uint32_t div = grouped ? 4 : 1;  // grouped: one box per four 32-column atoms
  const uint32_t bn = co_tile_n(co);
  const double tiles_n = double((ncols + kTcBM - 1) / kTcBM) * ((co + bn - 1) / bn);
  const double tiles_m = double((co + kTcBM - 1) / kTcBM) * ((ncols + kPBN - 1) / kPBN);
  const double on_n =
      tiles_n * stage_cycles(krows / 8, bn, kTcBM / 32 / div + 1,
                             (kTcBM / 32) * in_rows + w_rows_per_128 * bn / kTcBM);
  const double on_m =
      tiles_m * stage_cycles(krows / 8, kPBN, kPBN / 32 / div + 1,
                             (kPBN / 32) * in_rows + w_rows_per_128);
  return on_n <= on_m;
}

// CI / WIN orientation (measured better than the stage model above for
// conv2-5, whose channels-on-N epilogue stores and stream-K adds are scalar):
// the orientation with more useful flops per operand byte.
//   channels on M: 128 x 256 tile, operands (128 + 256) rows, useful co / 128-padded
//   channels on N: 128 x bn tile,  operands (128 + bn) rows,  useful co / bn-padded
bool choose_co_on_n_traffic(uint32_t co) {
  const double mt = (co + kTcBM - 1) / kTcBM * double(kTcBM);
  const double on_m = co / mt * (kTcBM * double(kPBN)) / (kTcBM + kPBN);
  const uint32_t bn = co_tile_n(co);
  const double nt = (co + bn - 1) / bn * double(bn);
  const double on_n = co / nt * (kTcBM * double(bn)) / (kTcBM + bn);
  return on_n > on_m * 1.02;
}

// channel rows of a ROW-mode filter image: tiles of co_tile_n (channels on
// N) or of 128 (channels on M)
uint32_t pack_rows(uint32_t co, bool co_on_n) {
  const uint32_t t = co_on_n ? co_tile_n(co) : kTcBM;
  return (co + t - 1) / t * t;
}

struct TcPlan {
  bool ok = false;
  ConvGeomTc g{};
  uint32_t K = 0;  // packed K (multiple of 32)
};

cudaError_t launch_conv_nchw_tc(const ConvArgs& a, const float* wpack, uint32_t Kp,
                               cudaStream_t s) {
  const uint32_t K = a.ci * a.fh * a.fw;
  NchwConvParams prm;
  if (!make_tmap_2d(&prm.a, wpack, Kp, a.co, static_cast<uint64_t>(Kp) * 4, kTcBK, kTcBM, false))
    return cudaErrorInvalidValue;
  prm.x = a.src;
  prm.y = a.dst;
  prm.Ci = a.ci;
  prm.H = a.h;
  prm.W = a.w;
  prm.Co = a.co;
  prm.FH = a.fh;
  prm.FW = a.fw;
  prm.S = a.stride;
  prm.Pad = a.pad;
  prm.Ho = a.ho;
  prm.Wo = a.wo;
  prm.P = a.ho * a.wo;
  prm.K = K;
  prm.kb = Kp / kTcBK;
  prm.ncols = a.n * prm.P;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_nchw_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kTcSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid((prm.ncols + kTcBN - 1) / kTcBN, (a.co + kTcBM - 1) / kTcBM);
  lcnn_pdl::launch(tc_conv_nchw_kernel, grid, kNchwThreads, kTcSmem, s, prm);
  return cudaGetLastError();
}

TcPlan plan_tc(uint32_t n, uint32_t ci, uint32_t h, uint32_t w, int layout, uint32_t co,
               uint32_t fh, uint32_t fw, uint32_t stride, uint32_t pad, uint32_t ho,
               uint32_t wo) {
  TcPlan p;
  if (layout != LCNN_CHWN || n % 32 != 0) return p;
  ConvGeomTc& g = p.g;
  g = ConvGeomTc{n, ci, h, w, co, fh, fw, stride, pad, ho, wo, 0, 0, 0, 0};
  const uint64_t ncols = static_cast<uint64_t>(ho) * wo * n;
  if (ncols >= (1ull << 31) || static_cast<uint64_t>(h) * w * n * ci >= (1ull << 32)) return p;
  // padded K of the two small-channel packings
  const uint32_t kr = (ci * fw + 7) / 8 * 8;                   // ROW
  const uint32_t fp = fw <= 4 ? 4 : (fw <= 8 ? 8 : 16), cib = 32 / fp;
  const uint32_t win_k = fw <= 16 ? fh * ((ci + cib - 1) / cib * cib) * fp : ~0u;  // WIN
  if (ci % 32 == 0) {
    g.mode = kModeCI;
    p.K = fh * fw * ci;
  } else if (kr <= 64 && fh * kr < win_k) {
    g.mode = kModeROW;
    g.KR = kr;
    g.FP = fw;
    if (n % 128 == 0) {  // grouped input boxes: rows per group a multiple of 8
      uint32_t wb = fw;
      while ((ci * wb) % 8) ++wb;
      if (ci * wb <= 64) {
        g.FP = wb;
        g.KR = ci * wb;
      }
    }
    p.K = fh * g.KR;
  } else if (fw <= 16) {
    g.mode = kModeWIN;
    g.FP = fp;
    g.CIB = cib;
    g.CiP = (ci + g.CIB - 1) / g.CIB * g.CIB;
    p.K = fh * g.CiP * g.FP;
  } else {
    return p;
  }
  p.ok = true;
  return p;
}

}  // namespace

struct ConvTcArgs {
  const ConvArgs& a;
  const TcPlan& p;
  const float *w_hi, *w_lo, *x_hi, *x_lo;
};

// Zero the stream-K region of out[co][col] (whole tiles inside it are
// overwritten by plain stores anyway).  co_on_n: tile rows are columns.
// With a caller-owned sync word (ConvArgs::zsync) the persistent kernel
// zeroes the region itself (Sched::zsync); pass sync = nullptr for kernels
// that do not implement it.
cudaError_t zero_sk_region(Sched& sc, bool co_on_n, uint32_t bw, float* dst, uint32_t ncols,
                           uint32_t co, cudaStream_t s, uint32_t tm = kTcBM,
                           unsigned long long* sync = nullptr) {
  if (sc.dp_tiles >= sc.mt * sc.nt) return cudaSuccess;
  const uint32_t nt0 = sc.dp_tiles / sc.mt;
  uint32_t row0, col0;
  if (co_on_n) {
    row0 = nt0 * bw;
    col0 = nt0 == sc.nt - 1 ? (sc.dp_tiles % sc.mt) * tm : 0;
  } else {
    row0 = 0;
    col0 = nt0 * kPBN;
  }
  return sched_zero_region(sc, sync, dst + uint64_t{row0} * ncols + col0, ncols, ncols - col0,
                           co - row0, nt0 * sc.mt,
                           [s](float* p, uint64_t pitch, uint64_t width, uint64_t rows) {
                             return launch_zero2d(p, pitch, width, rows, s);
                           });
}

template <bool kCoOnN>
cudaError_t launch_chwn_row(const ConvTcArgs& t, cudaStream_t s, bool rows2 = false) {
  const ConvArgs& a = t.a;
  const TcPlan& p = t.p;
  const uint32_t kr = p.g.KR, bn = kCoOnN ? co_tile_n(a.co) : kTcBM;  // filter tile rows
  ChwnRowLoader<kCoOnN> L;
  L.wimg[0] = t.w_hi;
  L.wimg[1] = t.w_lo;
  const uint64_t dims[4] = {a.n, a.w, a.h, a.ci};
  const uint64_t pitch[3] = {static_cast<uint64_t>(a.n) * 4, static_cast<uint64_t>(a.w) * a.n * 4,
                             static_cast<uint64_t>(a.h) * a.w * a.n * 4};
  L.grouped = a.n % 128 == 0 && p.g.KR == a.ci * p.g.FP;
  if (L.grouped) {
    const uint64_t gdims[5] = {32, a.w, a.ci, a.n / 32, a.h};
    const uint64_t gpitch[4] = {pitch[0], pitch[2], 128, pitch[1]};
    const uint32_t gbox[5] = {32, p.g.FP, a.ci, 4, 1};
    if (!make_tmap(&L.x[0], t.x_hi, 5, gdims, gpitch, gbox, nullptr, 1) ||
        !make_tmap(&L.x[1], t.x_lo, 5, gdims, gpitch, gbox, nullptr, 1))
      return cudaErrorInvalidValue;
  } else {
    const uint32_t box[4] = {32, a.fw, 1, a.ci};
    if (!make_tmap(&L.x[0], t.x_hi, 4, dims, pitch, box, nullptr, 1) ||
        !make_tmap(&L.x[1], t.x_lo, 4, dims, pitch, box, nullptr, 1))
      return cudaErrorInvalidValue;
  }
  L.g = p.g;
  L.rows2 = rows2 && !kCoOnN;
  const uint32_t span = a.wo * a.n;  // columns of one output row
  L.ncols = L.rows2 ? (a.ho + 1) / 2 * span : a.ho * span;
  if (L.rows2) L.g.FH = a.fh + 1;  // input rows per row pair
  L.bn = bn;
  const bool x3 = a.precision == LCNN_PREC_3XTF32;
  const uint32_t ctiles = (a.co + bn - 1) / bn;
  Sched sc = kCoOnN ? make_sched((L.ncols + kTcBM - 1) / kTcBM, ctiles, a.fh, x3 ? 3 : 1, bn,
                                 true, false)
                    : make_sched(ctiles, (L.ncols + kPBN - 1) / kPBN, L.g.FH, x3 ? 3 : 1, kPBN,
                                 false, true);
  const uint32_t x_region = L.kBoxes * kr * 128;                  // input groups of KR rows
  const uint32_t in_bytes = L.kBoxes * a.ci * (L.grouped ? p.g.FP : a.fw) * 128;  // TMA bytes
  const uint32_t w_region = bn * kr * 4;                          // one filter row of the tile
  sc.ksteps = kr / 8;
  // resident filter image (channels on N): one channel tile, one segment,
  // >= 3 ring slots; LCNN_TC_PROBE bit 4 disables it
  const uint32_t img = a.fh * w_region;
  uint32_t slots = 0;
  if (kCoOnN && !x3 && sc.nt == 1 && !(sc.probe & 4))
    for (uint32_t n = kPStages; n >= 3 && !slots; --n)
      if (1024 + n * x_region + img + 16 + sizeof(PCtl) <= kMaxDynSmem) slots = n;
  if (slots) {
    L.res = img;
    sc.a_bytes = x_region;
    sc.stage_bytes = in_bytes;
    sched_ring(sc, slots, x_region, img);
  } else {
    L.res = 0;
    sc.a_bytes = kCoOnN ? x_region : w_region;
    sc.stage_bytes = in_bytes + w_region;
    const uint32_t stride = (x_region + w_region + 1023) / 1024 * 1024;
    uint32_t n = kPStages;
    const uint32_t epi = kCoOnN ? 0 : 1024 + kEpiStageBytes;  // RowsOut TMA-store staging
    while (n > 2 && 1024 + n * stride + epi + 16 + sizeof(PCtl) > kMaxDynSmem) --n;
    sched_ring(sc, n, stride, 0);
  }
  if (L.rows2) {
    if (sc.dp_tiles < sc.mt * sc.nt) {
      // split tiles: zero every output row from the first split row pair on
      // (tiles from the first one touching that pair wait for it)
      const uint32_t pr0 = static_cast<uint32_t>(uint64_t{sc.dp_tiles / sc.mt} * kPBN / span);
      const uint64_t ncols = uint64_t{a.ho} * span, col0 = uint64_t{2 * pr0} * span;
      // blocked output: from pixel col0 / N on, in each of the N/32 groups
      const bool blk = a.blk & LCNN_CONV_OUT_HWCN32;
      const uint64_t hw = uint64_t{a.ho} * a.wo, px0 = col0 / a.n, run = uint64_t{a.co} * 32;
      cudaError_t e = sched_zero_region(
          sc, a.zsync, blk ? a.dst + px0 * run : a.dst + col0, blk ? hw * run : ncols,
          blk ? (hw - px0) * run : ncols - col0, blk ? a.n / 32 : a.co,
          static_cast<uint32_t>(uint64_t{pr0} * span / kPBN) * sc.mt,
          [s](float* z, uint64_t pitch, uint64_t width, uint64_t rows) {
            return launch_zero2d(z, pitch, width, rows, s);
          });
      if (e != cudaSuccess) return e;
    }
    static const int pairs = [] {  // profiling knob LCNN_ROW2_PAIRS: 0 one box per fence,
      const char* e = std::getenv("LCNN_ROW2_PAIRS");  // 2 per-lane stores (no TMA),
      return e ? std::atoi(e) : 3;                      // 1 paired boxes, 3 quad boxes
    }();
    if (pairs == 3 && span % 128 == 0) {
      // quad boxes: 64 KB of staging; the ring gives up slots for it
      Sched se = sc;
      uint32_t n = se.stages;
      while (n > 2 && 1024 + n * se.stage_stride + 1024 + 4 * 4 * 4096 + 16 + sizeof(PCtl) >
                          kMaxDynSmem)
        --n;
      if (1024 + n * se.stage_stride + 1024 + 4 * 4 * 4096 + 16 + sizeof(PCtl) <= kMaxDynSmem) {
        sched_ring(se, n, se.stage_stride, 0);
        sched_epi(se, 0, 4);
        RowsQuadOut O;
        O.c = a.dst;
        O.ldc = uint64_t{a.ho} * span;
        O.M = a.co;
        O.span = span;
        O.ho = a.ho;
        const uint64_t dims[2] = {uint64_t{a.ho} * span, a.co};
        const uint64_t opitch[1] = {dims[0] * 4};
        const uint32_t obox[2] = {32, 32};
        const uint64_t qdims[3] = {32, dims[0] / 32, a.co};
        const uint64_t qpitch[2] = {128, dims[0] * 4};
        const uint32_t qbox[3] = {32, 4, 32};
        if (a.blk & LCNN_CONV_OUT_HWCN32) {  // 4D views {32 i, N/32, Ho*Wo, C}
          O.nimg = a.n;
          O.hw = a.ho * a.wo;
          const uint64_t bdims[4] = {32, a.n / 32, uint64_t{O.hw}, a.co};
          const uint64_t bpitch[3] = {uint64_t{O.hw} * a.co * 128, uint64_t{a.co} * 128, 128};
          const uint32_t cbox[4] = {32, 1, 1, 32}, bqbox[4] = {32, 4, 1, 32};
          if (a.n % 128 || !make_tmap(&O.y, a.dst, 4, bdims, bpitch, cbox, nullptr, 0) ||
              !make_tmap(&O.yq, a.dst, 4, bdims, bpitch, bqbox, nullptr, 0))
            return cudaErrorInvalidValue;
        } else if (!make_tmap(&O.y, a.dst, 2, dims, opitch, obox, nullptr, 0) ||
                   !make_tmap(&O.yq, a.dst, 3, qdims, qpitch, qbox, nullptr, 0)) {
          return cudaErrorInvalidValue;
        }
        return launch_persistent(L, O, se, s);
      }
    }
    if (a.blk) return cudaErrorNotSupported;  // the blocked output needs the quad epilogue
    if (pairs == 2) {
      RowsPairOutT<false, false> O{a.dst, uint64_t{a.ho} * span, a.co, span, a.ho};
      return launch_persistent(L, O, sc, s);
    }
    const uint64_t dims[2] = {uint64_t{a.ho} * span, a.co};
    const uint64_t opitch[1] = {dims[0] * 4};
    const uint32_t obox[2] = {32, 32};
    Sched se = sc;
    sched_epi(se, 0);
    if (pairs) {
      RowsPairOutT<true> O{a.dst, uint64_t{a.ho} * span, a.co, span, a.ho};
      if (!make_tmap(&O.y, a.dst, 2, dims, opitch, obox, nullptr, 0)) return cudaErrorInvalidValue;
      return launch_persistent(L, O, se, s);
    }
    RowsPairOutT<false> O{a.dst, uint64_t{a.ho} * span, a.co, span, a.ho};
    if (!make_tmap(&O.y, a.dst, 2, dims, opitch, obox, nullptr, 0)) return cudaErrorInvalidValue;
    return launch_persistent(L, O, se, s);
  }
  if (cudaError_t e = zero_sk_region(sc, kCoOnN, kCoOnN ? bn : kTcBM, a.dst, L.ncols, a.co, s,
                                     kTcBM, a.zsync);
      e != cudaSuccess)
    return e;
  if constexpr (kCoOnN) {
    ColsOutPlain O{a.dst, L.ncols, a.co};
    return launch_persistent(L, O, sc, s);
  } else {
    RowsOut O{a.dst, L.ncols, a.co, L.ncols};
    O.keep_l2 = keep_l2_knob() >= 2;
    if (!make_rows_out_map(&O.y, O)) return cudaErrorInvalidValue;
    Sched se = sc;
    sched_epi(se, 0);  // RowsOut never has a resident operand
    return launch_persistent(L, O, se, s);
  }
}

// SHARE-mode geometry: filter image rows, input box width, ring slot
// layout [filter row (A) | input box rows (B)] and how many slots fit.
// resident (profiling knob LCNN_CONV_ROW=r): the whole filter image stays in
// shared memory and slots carry only the input box.
struct ShareGeom {
  uint32_t bn, kr, bw, wbytes, slot, img, slots;
  bool ok;
};

// TMA-store staging boxes per epilogue warp in SHARE mode (profiling knob
// LCNN_SHARE_EPI=1: one box, a deeper input ring)
uint32_t share_epi_bufs() {
  static const uint32_t b = [] {
    const char* e = std::getenv("LCNN_SHARE_EPI");
    return e && e[0] == '1' ? 1u : 2u;
  }();
  return b;
}

ShareGeom share_geom(const ConvArgs& a, bool resident) {
  ShareGeom q{};
  q.bn = (a.co + 7) / 8 * 8;
  q.kr = (a.ci * a.fw + 7) / 8 * 8;
  q.bw = a.stride * (kSharePix - 1) + a.fw;
  const uint32_t rows = std::max(q.bw * a.ci, a.stride * a.ci * (kSharePix - 1) + q.kr);
  q.wbytes = resident ? 0 : q.kr * q.bn * 4;  // one filter row (a multiple of 128 B)
  q.slot = (q.wbytes + rows * 128 + 1023) / 1024 * 1024;
  q.img = resident ? a.fh * q.kr * q.bn * 4 + 16 * 128 : 0;  // + slack for the M = 128 reads
  q.slots = 0;
  for (uint32_t n = kPStagesMax; n >= 3 && !q.slots; --n)
    if (1024ull + n * q.slot + q.img + 1024 + share_epi_bufs() * 4 * 4096 + sizeof(PCtl) <=
        kMaxDynSmem)
      q.slots = n;
  q.ok = a.precision == LCNN_PREC_TF32 && a.co <= kTcBM && a.n % 32 == 0 && a.ci <= 256 &&
         q.bw <= 256 && q.kr <= 256 && a.stride * a.ci * 128 < (1u << 18) && q.slots >= 3;
  return q;
}

// Output view of the ShareOut TMA-store epilogue (see ShareOut::y).
bool make_share_out_map(CUtensorMap* m, const ConvArgs& a) {
  const uint64_t dims[5] = {32, a.n / 32, a.wo, a.ho, a.co};
  const uint64_t pitch[4] = {128, static_cast<uint64_t>(a.n) * 4,
                             static_cast<uint64_t>(a.wo) * a.n * 4,
                             static_cast<uint64_t>(a.ho) * a.wo * a.n * 4};
  const uint32_t box[5] = {32, 1, 1, 1, 32};
  return make_tmap(m, a.dst, 5, dims, pitch, box, nullptr, 0);
}

cudaError_t launch_chwn_share(const ConvTcArgs& t, bool resident, cudaStream_t s) {
  const ConvArgs& a = t.a;
  const ShareGeom q = share_geom(a, resident);
  ChwnShareLoader L;
  L.g = t.p.g;
  L.bn = q.bn;
  L.wimg = t.w_hi;
  L.owb = (a.wo + kSharePix - 1) / kSharePix;
  L.groups = a.n / 32;
  L.res = resident ? a.fh * q.kr * q.bn * 4 : 0;
  const uint64_t dims[5] = {32, a.ci, a.w, a.n / 32, a.h};
  const uint64_t pitch[4] = {static_cast<uint64_t>(a.h) * a.w * a.n * 4,
                             static_cast<uint64_t>(a.n) * 4, 128,
                             static_cast<uint64_t>(a.w) * a.n * 4};
  const uint32_t box[5] = {32, a.ci, q.bw, 1, 1};
  if (!make_tmap(&L.x, t.x_hi, 5, dims, pitch, box, nullptr, 1)) return cudaErrorInvalidValue;
  const uint32_t tiles = a.ho * L.owb * L.groups;
  Sched sc = make_sched(1, tiles, a.fh, 1, kSharePix * 32, false, true);
  sc.ksteps = q.kr / 8;
  sc.a_bytes = q.wbytes;
  sc.stage_bytes = q.wbytes + q.bw * a.ci * 128;
  sched_ring(sc, q.slots, q.slot, q.img);
  sched_epi(sc, q.img, share_epi_bufs());
  if (sc.dp_tiles < tiles) {  // zero the stream-K tiles' output rows (oh >= first split row)
    const uint64_t ncols = static_cast<uint64_t>(a.ho) * a.wo * a.n;
    const uint64_t col0 = static_cast<uint64_t>(sc.dp_tiles / (L.owb * L.groups)) * a.wo * a.n;
    cudaError_t e = launch_zero2d(a.dst + col0, ncols, ncols - col0, a.co, s);
    if (e != cudaSuccess) return e;
  }
  ShareOut O{a.dst, static_cast<uint64_t>(a.ho) * a.wo * a.n, a.co, a.n, a.wo, L.owb, L.groups};
  if (!make_share_out_map(&O.y, a)) return cudaErrorInvalidValue;
  O.fd_groups = FastDiv(L.groups);
  O.fd_owb = FastDiv(L.owb);
  return launch_persistent(L, O, sc, s);
}

// SHARE convolution + stride-2 max pooling (PWIN = 2 or 3) in one kernel
// (SharePoolOut).  Units = pooling strips (32-image group x PC pool
// columns) x row segments, one CTA each, so no split tiles and no zeroing.
template <int PWIN, bool kDirect>
cudaError_t launch_chwn_share_pool(const ConvTcArgs& t, float* pooled, uint32_t hp, uint32_t wp,
                                   cudaStream_t s) {
  using D = SharePoolDims<PWIN>;
  const ConvArgs& a = t.a;
  const ShareGeom q = share_geom(a, false);
  ChwnSharePoolLoader L;
  L.g = t.p.g;
  L.bn = q.bn;
  L.wimg = t.w_hi;
  L.groups = a.n / 32;
  L.owb = 0;
  L.res = 0;
  L.tpx = D::TPX;
  L.pc = D::PC;
  L.hp = hp;
  const uint32_t bw = a.stride * (D::TPX - 1) + a.fw;
  const uint64_t dims[5] = {32, a.ci, a.w, a.n / 32, a.h};
  const uint64_t pitch[4] = {static_cast<uint64_t>(a.h) * a.w * a.n * 4,
                             static_cast<uint64_t>(a.n) * 4, 128,
                             static_cast<uint64_t>(a.w) * a.n * 4};
  const uint32_t box[5] = {32, a.ci, bw, 1, 1};
  if (!make_tmap(&L.x, t.x_hi, 5, dims, pitch, box, nullptr, 1)) return cudaErrorInvalidValue;
  const uint32_t jc = (wp + D::PC - 1) / D::PC;
  L.strips = L.groups * jc;
  const uint32_t sms = static_cast<uint32_t>(tc_sm_count());
  L.segs = std::max(1u, std::min(hp, sms / L.strips));
  L.units = L.strips * L.segs;
  uint32_t rmax = 0;
  for (uint32_t sg = 0; sg < L.segs; ++sg)
    rmax = std::max(rmax, 2 * ((sg + 1) * hp / L.segs - sg * hp / L.segs) + PWIN - 2);
  L.fd_units = FastDiv(L.units);
  L.fd_groups = FastDiv(L.groups);
  Sched sc = make_sched(1, L.units * rmax, a.fh, 1, D::TPX * 32, false, true, kMinSkIters, L.units);
  if (sc.dp_tiles != L.units * rmax || sc.grid != L.units) return cudaErrorInvalidConfiguration;
  sc.ksteps = q.kr / 8;
  sc.a_bytes = q.wbytes;
  sc.stage_bytes = q.wbytes + bw * a.ci * 128;
  // slots: the ring of input boxes, after the staging boxes (2 per epilogue
  // warp, double-buffered TMA stores) unless the lanes store directly
  const uint32_t slot = (q.wbytes + std::max(bw * a.ci, a.stride * a.ci * (D::TPX - 1) + q.kr) * 128 +
                         1023) / 1024 * 1024;
  const uint32_t epi = kDirect ? 0u : 2u;
  uint32_t slots = 0;
  for (uint32_t n = kPStagesMax; n >= 3 && !slots; --n)
    if (1024ull + n * slot + 1024 + epi * 4 * 4096 + sizeof(PCtl) <= kMaxDynSmem) slots = n;
  if (!slots) return cudaErrorInvalidConfiguration;
  sched_ring(sc, slots, slot, 0);
  if (epi) sched_epi(sc, 0, epi);
  SharePoolOut<PWIN, kDirect> O;
  O.out = pooled;
  O.n = a.n;
  {
    const uint64_t odims[5] = {32, a.n / 32, wp, hp, a.co};
    const uint64_t opitch[4] = {128, static_cast<uint64_t>(a.n) * 4,
                                static_cast<uint64_t>(wp) * a.n * 4,
                                static_cast<uint64_t>(hp) * wp * a.n * 4};
    const uint32_t obox[5] = {32, 1, 1, 1, 32};
    if (!make_tmap(&O.y, pooled, 5, odims, opitch, obox, nullptr, 0))
      return cudaErrorInvalidValue;
  }
  O.co = a.co;
  O.wp = wp;
  O.hp = hp;
  O.strips = L.strips;
  O.segs = L.segs;
  O.fd_units = L.fd_units;
  O.fd_groups = L.fd_groups;
  return launch_persistent(L, O, sc, s);
}

// TAPS-mode geometry: input box width, ring slots that fit shared memory.
struct TapsGeom {
  uint32_t bw, ibox, islot, ni, nf;
  bool ok;
};

TapsGeom taps_geom(const ConvArgs& a, uint32_t reserve = 0) {
  TapsGeom q{};
  q.bw = a.stride * (kSharePix - 1) + a.fw;
  q.ibox = q.bw * 4096;
  q.islot = (q.ibox + 1023) / 1024 * 1024;
  const uint64_t avail = kMaxDynSmem - 1024 - sizeof(TapsCtl) - 16 - reserve;
  // input-box slots: 3 (profiling knob LCNN_TAPS_NI = 2..4 tries other rings;
  // fewer input slots leave more filter slots)
  static const uint32_t ni_max = [] {
    const char* e = std::getenv("LCNN_TAPS_NI");
    const int v = e ? std::atoi(e) : 3;
    return static_cast<uint32_t>(v < 2 ? 2 : (v > 4 ? 4 : v));
  }();
  for (uint32_t ni = ni_max; ni >= 2 && !q.ni; --ni) {
    if (ni * uint64_t{q.islot} >= avail) continue;
    const uint64_t nf = std::min<uint64_t>(8, (avail - ni * uint64_t{q.islot}) / kTcABytes);
    if (nf >= std::max<uint64_t>(4, a.fw + 1)) {
      q.ni = ni;
      q.nf = static_cast<uint32_t>(nf);
    }
  }
  q.ok = a.precision == LCNN_PREC_TF32 && a.ci % 32 == 0 && a.n % 32 == 0 && q.bw <= 256 &&
         q.ni >= 2 && a.stride * 4096u < (1u << 18);
  return q;
}

cudaError_t launch_chwn_taps(const ConvTcArgs& t, cudaStream_t s, bool rows2 = false,
                             float* pooled = nullptr, uint32_t hp = 0, uint32_t wp = 0) {
  const ConvArgs& a = t.a;
  // TMA-store epilogue for row pairs (measured on B200, VGG conv1_2 1461 -> 1450 us; slower on
  // the C_o = 128 layers: conv2_1 534 -> 577, conv2_2 949 -> 984 us, whose per-lane stores
  // overlap better; profiles/r02_taps_tma_ab.jsonl).  Profiling knob LCNN_TAPS_TMA = 0 off,
  // 1 row pairs only (default), 2 always.
  static const int tma_knob = [] {
    const char* e = std::getenv("LCNN_TAPS_TMA");
    return e ? std::atoi(e) : 1;
  }();
  const bool pool = pooled != nullptr;  // the 2x2 max pool in the epilogue (rows2 only)
  if (pool && !rows2) return cudaErrorInvalidValue;
  const bool tma = pool || tma_knob == 2 || (tma_knob == 1 && rows2);
  constexpr uint32_t kEpi = 4 * 2 * 4096;
  TapsGeom q = taps_geom(a, tma ? kEpi + 1024 : 0);
  if (!q.ok) q = taps_geom(a);
  TapsParams prm;
  prm.rows2 = rows2 ? 1u : 0u;
  prm.Ho = a.ho;
  prm.tma = tma && q.ok && taps_geom(a, kEpi + 1024).ok ? 1u : 0u;
  if (pool && !prm.tma) return cudaErrorInvalidConfiguration;  // no room for the staging
  prm.pool_out = pooled;
  prm.pool = pool ? 1u : 0u;
  prm.hp = hp;
  prm.wp = wp;
  const uint64_t dims[5] = {32, a.ci, a.w, a.n / 32, a.h};
  uint64_t pitch[4] = {static_cast<uint64_t>(a.h) * a.w * a.n * 4,
                       static_cast<uint64_t>(a.n) * 4, 128,
                       static_cast<uint64_t>(a.w) * a.n * 4};
  if (a.blk & LCNN_CONV_IN_HWCN32) {  // [N/32][H][W][C][32]: strides of c, w, g, h
    // (the box {32 n, 32 c, BW w} lands in shared memory exactly as from CHWN;
    // in HBM it is BW runs of 4 KB: 11.6 against 4.6 TB/s DRAM-cold,
    // profiles/r02_tma_bench_blocked_layouts.txt)
    pitch[0] = 128;
    pitch[1] = uint64_t{a.ci} * 128;
    pitch[2] = uint64_t{a.h} * a.w * a.ci * 128;
    pitch[3] = uint64_t{a.w} * a.ci * 128;
  }
  const uint32_t box[5] = {32, 32, q.bw, 1, 1};
  if (!make_tmap(&prm.x, t.x_hi, 5, dims, pitch, box, nullptr, 1)) return cudaErrorInvalidValue;
  const uint64_t K = t.p.K;
  if (!make_tmap_2d(&prm.w, t.w_hi, K, rows2 ? kTcBM : a.co, K * 4, kTcBK, kTcBM, false))
    return cudaErrorInvalidValue;
  prm.FW = a.fw;
  prm.S = a.stride;
  prm.P = a.pad;
  prm.CB = a.ci / 32;
  prm.OWB = (a.wo + kSharePix - 1) / kSharePix;
  prm.G = a.n / 32;
  prm.ni = q.ni;
  prm.nf = q.nf;
  prm.islot = q.islot;
  prm.ibox = q.ibox;
  const uint32_t rows = rows2 ? (a.ho + 1) / 2 : a.ho;  // tile rows (row pairs)
  const uint32_t mt = rows2 ? 1 : (a.co + kTcBM - 1) / kTcBM, nt = rows * prm.OWB * prm.G;
  prm.sc = make_sched(mt, nt, (a.fh + prm.rows2) * prm.CB, 1, kSharePix * 32, false, true);
  if (pool) {  // whole tiles only: a window needs the finished sums of its tile
    Sched& z = prm.sc;
    z.dp_tiles = mt * nt;
    z.sk_iters = 0;
    z.sk_ctas = 0;
    z.grid = std::min<uint32_t>(z.dp_tiles, static_cast<uint32_t>(tc_sm_count()));
  }
  prm.ctl_off = q.ni * q.islot + q.nf * kTcABytes;
  prm.epi_off = 0;
  if (prm.tma) {
    prm.epi_off = (prm.ctl_off + 1023) / 1024 * 1024;
    prm.ctl_off = prm.epi_off + kEpi;
    prm.sc.epi_bufs = 2;
  }
  prm.out = ShareOut{a.dst, static_cast<uint64_t>(a.ho) * a.wo * a.n, a.co, a.n, a.wo, prm.OWB,
                     prm.G};
  if (prm.tma && !pool) {
    if (!make_share_out_map(&prm.out.y, a)) return cudaErrorInvalidValue;
    prm.out.fd_groups = FastDiv(prm.G);
    prm.out.fd_owb = FastDiv(prm.OWB);
  }
  // L2 policies (profiling knob LCNN_TAPS_L2, bit 1: input boxes evict_last,
  // bit 2: TMA-stored outputs evict_first)
  static const int l2_knob = [] {
    const char* e = std::getenv("LCNN_TAPS_L2");
    return e ? std::atoi(e) : 0;
  }();
  prm.in_keep = (l2_knob & 1) ? 1u : 0u;
  prm.out.evict_first = (l2_knob & 2) ? 1u : 0u;
  const Sched& sc = prm.sc;
  if (sc.dp_tiles < mt * nt) {  // zero the stream-K tiles' output rows (oh >= first split row)
    const uint64_t ncols = static_cast<uint64_t>(a.ho) * a.wo * a.n;
    const uint32_t r0 = sc.dp_tiles / mt / (prm.OWB * prm.G);  // first split tile row
    const uint64_t col0 = (static_cast<uint64_t>(r0) << prm.rows2) * a.wo * a.n;
    cudaError_t e = sched_zero_region(prm.sc, a.zsync, a.dst + col0, ncols, ncols - col0, a.co,
                                      r0 * prm.OWB * prm.G * mt,
                                      [s](float* z, uint64_t pitch, uint64_t width, uint64_t rows) {
                                        return launch_zero2d(z, pitch, width, rows, s);
                                      });
    if (e != cudaSuccess) return e;
  }
  const uint32_t smem = 1024 + prm.ctl_off + static_cast<uint32_t>(sizeof(TapsCtl));
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_taps_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return lcnn_pdl::launch(tc_conv_taps_kernel, sc.grid, kTcThreads, smem, s, prm);
}

// TAPS with two accumulators (tc_conv_taps_acc2_kernel): a TAPS-routed layer
// (not the C_o <= 64 row pairs) at stride 1 with >= 2 output rows.
// Profiling knob LCNN_TAPS_ACC2=0: one output row per tile.
bool taps_acc2_ok(const ConvArgs& a) {
  static const bool on = [] {
    const char* e = std::getenv("LCNN_TAPS_ACC2");
    return !(e && e[0] == '0');
  }();
  return on && a.stride == 1 && a.ho >= 2 && a.precision == LCNN_PREC_TF32;
}

cudaError_t launch_chwn_taps_acc2(const ConvTcArgs& t, cudaStream_t s, float* pooled = nullptr,
                                  uint32_t hp = 0, uint32_t wp = 0) {
  const ConvArgs& a = t.a;
  const bool pool = pooled != nullptr;
  constexpr uint32_t kPoolStg = 4 * 4 * 4096;  // 16 KB per epilogue warp
  const TapsGeom q = taps_geom(a, pool ? kPoolStg + 1024 : 0);
  if (!q.ok || a.stride != 1) return cudaErrorInvalidConfiguration;
  TapsParams prm{};
  const uint64_t dims[5] = {32, a.ci, a.w, a.n / 32, a.h};
  const uint64_t pitch[4] = {static_cast<uint64_t>(a.h) * a.w * a.n * 4,
                             static_cast<uint64_t>(a.n) * 4, 128,
                             static_cast<uint64_t>(a.w) * a.n * 4};
  const uint32_t box[5] = {32, 32, q.bw, 1, 1};
  if (!make_tmap(&prm.x, t.x_hi, 5, dims, pitch, box, nullptr, 1)) return cudaErrorInvalidValue;
  const uint64_t K = t.p.K;
  if (!make_tmap_2d(&prm.w, t.w_hi, K, a.co, K * 4, kTcBK, kTcBM, false))
    return cudaErrorInvalidValue;
  prm.FW = a.fw;
  prm.S = 1;
  prm.P = a.pad;
  prm.CB = a.ci / 32;
  prm.OWB = (a.wo + kSharePix - 1) / kSharePix;
  prm.G = a.n / 32;
  prm.ni = q.ni;
  prm.nf = q.nf;
  prm.islot = q.islot;
  prm.ibox = q.ibox;
  prm.Ho = a.ho;
  prm.FH = a.fh;
  const uint32_t mt = (a.co + kTcBM - 1) / kTcBM, nt = (a.ho + 1) / 2 * prm.OWB * prm.G;
  prm.sc = make_sched(mt, nt, (a.fh + 1) * prm.CB, 1, kSharePix * 32, false, true);
  {  // whole tiles only
    Sched& z = prm.sc;
    z.dp_tiles = mt * nt;
    z.sk_iters = 0;
    z.sk_ctas = 0;
    z.grid = std::min<uint32_t>(z.dp_tiles, static_cast<uint32_t>(tc_sm_count()));
  }
  prm.ctl_off = q.ni * q.islot + q.nf * kTcABytes;
  prm.epi_off = 0;
  if (pool) {
    prm.epi_off = (prm.ctl_off + 1023) / 1024 * 1024;
    prm.ctl_off = prm.epi_off + kPoolStg;
  }
  prm.out = ShareOut{a.dst, static_cast<uint64_t>(a.ho) * a.wo * a.n, a.co, a.n, a.wo, prm.OWB,
                     prm.G};
  prm.pool_out = pooled;
  prm.pool = pool ? 1u : 0u;
  prm.hp = hp;
  prm.wp = wp;
  const uint32_t smem = 1024 + prm.ctl_off + static_cast<uint32_t>(sizeof(TapsCtl));
  if (smem > kMaxDynSmem) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_taps_acc2_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return lcnn_pdl::launch(tc_conv_taps_acc2_kernel, prm.sc.grid, kTcThreads, smem, s, prm);
}

// TAPS-N geometry (tc_conv_tapsn_pair_kernel): C_o tile, input box width,
// ring slots that fit next to the 16 KB epilogue staging.
struct TapsNGeom {
  uint32_t bw, bwid, ibox, fslot, ni, nf;
  bool ok;
};

TapsNGeom tapsn_geom(const ConvArgs& a) {
  TapsNGeom q{};
  q.bw = co_tile_n(a.co);
  q.bwid = a.stride * (kTapsNPix - 1) + a.fw;
  q.ibox = q.bwid * 4096;
  q.fslot = q.bw / 2 * 128;
  const uint64_t avail = kMaxDynSmem - 1024 - 4 * 4096 - sizeof(TapsNCtl) - 16;
  for (uint32_t ni = 3; ni >= 2 && !q.ni; --ni) {
    if (ni * uint64_t{q.ibox} >= avail) continue;
    const uint64_t nf = std::min<uint64_t>(8, (avail - ni * uint64_t{q.ibox}) / q.fslot);
    if (nf >= std::max<uint64_t>(4, a.fw + 1)) {
      q.ni = ni;
      q.nf = static_cast<uint32_t>(nf);
    }
  }
  q.ok = a.precision == LCNN_PREC_TF32 && a.ci % 32 == 0 && a.n % 64 == 0 && q.bwid <= 256 &&
         q.bw % 32 == 0 && q.ni >= 2 && a.stride * 4096u < (1u << 18);
  return q;
}

cudaError_t launch_chwn_tapsn(const ConvTcArgs& t, cudaStream_t s) {
  const ConvArgs& a = t.a;
  const TapsNGeom q = tapsn_geom(a);
  TapsNParams prm;
  const uint64_t dims[5] = {32, a.ci, a.w, a.n / 32, a.h};
  const uint64_t pitch[4] = {static_cast<uint64_t>(a.h) * a.w * a.n * 4,
                             static_cast<uint64_t>(a.n) * 4, 128,
                             static_cast<uint64_t>(a.w) * a.n * 4};
  const uint32_t box[5] = {32, 32, q.bwid, 1, 1};
  if (!make_tmap(&prm.x, t.x_hi, 5, dims, pitch, box, nullptr, 1)) return cudaErrorInvalidValue;
  const uint64_t K = t.p.K;
  if (!make_tmap_2d(&prm.w, t.w_hi, K, a.co, K * 4, kTcBK, q.bw / 2, false))
    return cudaErrorInvalidValue;
  if (!make_share_out_map(&prm.y, a)) return cudaErrorInvalidValue;
  prm.FW = a.fw;
  prm.S = a.stride;
  prm.P = a.pad;
  prm.CB = a.ci / 32;
  prm.OWB = (a.wo + kTapsNPix - 1) / kTapsNPix;
  prm.G2 = a.n / 64;
  prm.Wo = a.wo;
  prm.bw = q.bw;
  prm.ni = q.ni;
  prm.nf = q.nf;
  prm.islot = q.ibox;
  prm.ibox = q.ibox;
  prm.fslot = q.fslot;
  prm.epi_off = q.ni * q.ibox + q.nf * q.fslot;  // 1 KB multiples
  prm.ctl_off = prm.epi_off + 4 * 4096;
  const uint32_t mt = (a.co + q.bw - 1) / q.bw, nt = a.ho * prm.OWB * prm.G2;
  // stream-K tail at any wave count (measured: VGG conv3_2 566 us with it,
  // 578 us whole-tile)
  prm.sc = make_sched(mt, nt, a.fh * prm.CB, 1, q.bw, true, false, kMinSkIters,
                      static_cast<uint32_t>(tc_sm_count() / 2), 0);
  prm.sc.idesc = idesc_tf32(2 * kTcBM, q.bw, true, false);
  prm.sc.grid *= 2;
  const Sched& sc = prm.sc;
  if (sc.dp_tiles < mt * nt) {  // zero the stream-K tiles' output rows (oh >= first split row)
    const uint64_t ncols = static_cast<uint64_t>(a.ho) * a.wo * a.n;
    const uint32_t r0 = sc.dp_tiles / mt / (prm.OWB * prm.G2);  // first split tile row
    const uint64_t col0 = static_cast<uint64_t>(r0) * a.wo * a.n;
    cudaError_t e = sched_zero_region(prm.sc, a.zsync, a.dst + col0, ncols, ncols - col0, a.co,
                                      r0 * prm.OWB * prm.G2 * mt,
                                      [s](float* z, uint64_t pitch, uint64_t width, uint64_t rows) {
                                        return launch_zero2d(z, pitch, width, rows, s);
                                      });
    if (e != cudaSuccess) return e;
  }
  const uint32_t smem = 1024 + prm.ctl_off + static_cast<uint32_t>(sizeof(TapsNCtl));
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_tapsn_pair_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (smem > kMaxDynSmem || sc.grid % 2) return cudaErrorInvalidConfiguration;
  return lcnn_pdl::launch(tc_conv_tapsn_pair_kernel, sc.grid, kTcThreads, smem, s, prm);
}

template <bool kCoOnN, bool kPair = false>
cudaError_t launch_chwn_tc(const ConvTcArgs& t, cudaStream_t s) {
  const ConvArgs& a = t.a;
  const TcPlan& p = t.p;
  const bool x3 = a.precision == LCNN_PREC_3XTF32;
  const uint32_t bw = kCoOnN ? co_tile_n(a.co) : kTcBM;  // filter tile rows
  const uint32_t wbox = kPair ? bw / 2 : bw;              // rows one CTA loads
  ChwnConvLoader<kCoOnN, kPair> L;
  const uint64_t K = p.K;
  if (!make_tmap_2d(&L.w[0], t.w_hi, K, a.co, K * 4, kTcBK, wbox, false) ||
      !make_tmap_2d(&L.w[1], t.w_lo, K, a.co, K * 4, kTcBK, wbox, false))
    return cudaErrorInvalidValue;
  const uint64_t dims[4] = {a.n, a.w, a.h, a.ci};
  const uint64_t pitch[3] = {static_cast<uint64_t>(a.n) * 4, static_cast<uint64_t>(a.w) * a.n * 4,
                             static_cast<uint64_t>(a.h) * a.w * a.n * 4};
  const uint32_t fp = p.g.mode == kModeCI ? 1 : p.g.FP, cib = p.g.mode == kModeCI ? 32 : p.g.CIB;
  L.grouped = a.n % 128 == 0;
  if (L.grouped) {
    const uint64_t gdims[5] = {32, a.w, a.ci, a.n / 32, a.h};
    const uint64_t gpitch[4] = {pitch[0], pitch[2], 128, pitch[1]};
    const uint32_t gbox[5] = {32, fp, cib, 4, 1};
    if (!make_tmap(&L.x[0], t.x_hi, 5, gdims, gpitch, gbox, nullptr, 1) ||
        !make_tmap(&L.x[1], t.x_lo, 5, gdims, gpitch, gbox, nullptr, 1))
      return cudaErrorInvalidValue;
  } else {
    const uint32_t box[4] = {32, fp, 1, cib};
    if (!make_tmap(&L.x[0], t.x_hi, 4, dims, pitch, box, nullptr, 1) ||
        !make_tmap(&L.x[1], t.x_lo, 4, dims, pitch, box, nullptr, 1))
      return cudaErrorInvalidValue;
  }
  L.g = p.g;
  L.ncols = a.ho * a.wo * a.n;
  const uint32_t segs = x3 ? 3 : 1;
  if constexpr (kPair) {
    // 256-column tiles on a CTA pair; per CTA a stage is its 128 input
    // columns (16 KB) + half the filter tile
    const uint32_t tm = 2 * kTcBM;
    Sched sc = make_sched((L.ncols + tm - 1) / tm, (a.co + bw - 1) / bw, p.K / kTcBK, segs, bw,
                          true, false, kMinSkIters, tc_sm_count() / 2);
    sc.idesc = idesc_tf32(tm, bw, true, false);
    sc.grid *= 2;
    sc.a_bytes = kTcABytes;
    sc.stage_bytes = kTcABytes + wbox * kTcBK * 4;
    const uint32_t stride = (sc.stage_bytes + 1023) / 1024 * 1024;
    uint32_t n = kPStagesMax;
    constexpr uint32_t epi = 1024 + 4 * 4096;  // one TMA-store box per epilogue warp
    while (n > 2 && 1024 + n * stride + epi + 16 + sizeof(PCtl) > kMaxDynSmem) --n;
    sched_ring(sc, n, stride, 0);
    sched_epi(sc, 0, 1);
    if (cudaError_t e = zero_sk_region(sc, true, bw, a.dst, L.ncols, a.co, s, tm); e != cudaSuccess)
      return e;
    ColsOut O{a.dst, L.ncols, a.co};
    O.keep_l2 = keep_l2_knob() >= 1;
    if (!make_cols_out_map(&O.y, O)) return cudaErrorInvalidValue;
    return launch_pair(L, O, sc, s);
  } else {
  Sched sc =
      kCoOnN ? make_sched((L.ncols + kTcBM - 1) / kTcBM, (a.co + bw - 1) / bw, p.K / kTcBK, segs,
                          bw, true, false)
             : make_sched((a.co + kTcBM - 1) / kTcBM, (L.ncols + kPBN - 1) / kPBN, p.K / kTcBK,
                          segs, kPBN, false, true);
  if (cudaError_t e = zero_sk_region(sc, kCoOnN, bw, a.dst, L.ncols, a.co, s, kTcBM, a.zsync);
      e != cudaSuccess)
    return e;
  if constexpr (kCoOnN) {
    ColsOut O{a.dst, L.ncols, a.co};
    if (!make_cols_out_map(&O.y, O)) return cudaErrorInvalidValue;
    Sched se = sc;
    sched_epi(se, 0);
    return launch_persistent(L, O, se, s);
  } else {
    RowsOut O{a.dst, L.ncols, a.co, L.ncols};
    O.keep_l2 = keep_l2_knob() >= 2;
    if (!make_rows_out_map(&O.y, O)) return cudaErrorInvalidValue;
    Sched se = sc;
    sched_epi(se, 0);
    return launch_persistent(L, O, se, s);
  }
  }
}

// ---- routing, filter packing and the packed launch ------------------------
// A convolution runs in two phases: the filters are packed into the operand
// image of the chosen kernel (once per weight set when the caller keeps the
// pack, e.g. a network layer), then the packed launch runs.  Packed image:
// [hi (apack floats) | lo (apack floats, 3xTF32 only)], each 256-B aligned.
// Run workspace (3xTF32 CHWN only): the split input copies [x_hi | x_lo].
namespace {

enum RouteKind { kRouteSimt, kRouteNchwTc, kRouteRowOnN, kRouteRowOnM, kRouteChwnOnN, kRouteChwnOnM,
                 kRouteShare, kRouteShareRes, kRouteChwnPair, kRouteTaps, kRouteTapsN,
                 kRouteTaps2, kRouteRowPairs };

struct ConvRoute {
  RouteKind kind = kRouteSimt;
  TcPlan p;
  uint64_t apack = 0;  // floats of one packed filter image
  uint32_t kp = 0;     // NCHW: K padded to the k-block
  // NCHW layer run as transpose -> the CHWN route `kind` -> transpose back
  // (the run workspace then also holds the CHWN input and output copies)
  bool via_chwn = false;
};

uint64_t align_floats(uint64_t f) { return (f + 63) / 64 * 64; }  // 256 B

ConvRoute route_conv(const ConvArgs& a) {
  ConvRoute r;
  // NCHW on the tensor cores: NCHW rows of odd width cannot be TMA tensors,
  // and the gather-producer kernel below reaches ~50 TF/s, so an NCHW layer
  // is run as NCHW->CHWN transpose (6+ TB/s), the CHWN route of the same
  // geometry, and CHWN->NCHW transpose of the output: AlexNet conv2 in NCHW
  // ~1.7 ms -> ~0.16 ms.  Profiling knob LCNN_CONV_NCHW=gather keeps the
  // gather kernel.
  static const bool nchw_gather = [] {
    const char* e = std::getenv("LCNN_CONV_NCHW");
    return e && e[0] == 'g';
  }();
  if (a.layout == LCNN_NCHW && a.precision != LCNN_PREC_FP32 && !nchw_gather &&
      static_cast<uint64_t>(a.n) * a.ci * a.h * a.w < (1ull << 32) &&
      static_cast<uint64_t>(a.n) * a.co * a.ho * a.wo < (1ull << 32)) {
    ConvArgs c = a;
    c.layout = LCNN_CHWN;
    ConvRoute inner = route_conv(c);
    if (inner.kind != kRouteSimt) {
      inner.via_chwn = true;
      return inner;
    }
  }
  if (a.layout == LCNN_NCHW && a.precision == LCNN_PREC_TF32 &&
      static_cast<uint64_t>(a.n) * a.ho * a.wo < (1ull << 31)) {
    r.kind = kRouteNchwTc;
    const uint32_t K = a.ci * a.fh * a.fw;
    r.kp = (K + kTcBK - 1) / kTcBK * kTcBK;
    r.apack = static_cast<uint64_t>(a.co) * r.kp;
    return r;
  }
  if (a.precision != LCNN_PREC_FP32)
    r.p = plan_tc(a.n, a.ci, a.h, a.w, a.layout, a.co, a.fh, a.fw, a.stride, a.pad, a.ho, a.wo);
  if (!r.p.ok) {
    r.kind = kRouteSimt;
    r.apack = static_cast<uint64_t>(a.co) * a.ci * a.fh * a.fw;  // the filters as given
    return r;
  }
  const uint64_t ncols = static_cast<uint64_t>(a.ho) * a.wo * a.n;
  if (r.p.g.mode == kModeROW) {
    // profiling knob LCNN_CONV_ROW: "n" / "m" force ROW mode in that
    // orientation instead of SHARE ("n" ungrouped, KR = C_i*F_w rounded to 8,
    // so the filter image can stay resident)
    static const int force = [] {
      const char* e = std::getenv("LCNN_CONV_ROW");
      return e ? (e[0] == 'n' ? 1 : (e[0] == 'm' ? 2 : (e[0] == 'r' ? 3 : 0))) : 0;
    }();
    // SHARE pays off with wide filter rows (AlexNet conv1, F_w = 11: 120 ->
    // 88 us against ROW); with F_w <= 3 a SHARE box saves little and ROW
    // with channels on M is faster (VGG conv1_1: 504 -> 446 us), so those
    // layers take ROW on M
    const bool narrow = !force && a.fw <= 3;
    if ((!force && !narrow) || force == 3) {
      const ShareGeom q = share_geom(a, force == 3);
      if (q.ok) {
        r.kind = force == 3 ? kRouteShareRes : kRouteShare;
        r.p.g.mode = kModeSHARE;
        r.p.g.KR = q.kr;
        r.p.g.FP = a.fw;
        r.p.K = a.fh * q.kr;
        r.apack = static_cast<uint64_t>(a.fh) * q.kr * q.bn;
        return r;
      }
    }
    if (force == 1) {
      r.p.g.KR = (a.ci * a.fw + 7) / 8 * 8;
      r.p.g.FP = a.fw;
      r.p.K = a.fh * r.p.g.KR;
    }
    const uint32_t kr = r.p.g.KR;
    const bool grouped = a.n % 128 == 0 && kr == a.ci * r.p.g.FP;
    bool on_n = choose_co_on_n(a.co, ncols, kr, grouped ? kr : a.ci * a.fw, kr * 4, grouped);
    if (force) on_n = force == 1;
    if (narrow) on_n = false;
    r.kind = on_n ? kRouteRowOnN : kRouteRowOnM;
    r.apack = static_cast<uint64_t>(pack_rows(a.co, on_n)) * r.p.K;
    // C_o <= 64 on M at stride 1: row pairs (output rows oh, oh + 1 on the
    // two halves of the 128-row MMA, F_h + 1 shared input rows; as TAPS row
    // pairs).  Profiling knob LCNN_CONV_ROW2=0 keeps one row per tile.
    static const bool row2_off = [] {
      const char* e = std::getenv("LCNN_CONV_ROW2");
      return e && e[0] == '0';
    }();
    if (!on_n && !row2_off && !force && a.co <= 64 && a.stride == 1 && a.ho >= 2 &&
        a.precision == LCNN_PREC_TF32) {
      r.kind = kRouteRowPairs;
      r.p.K = (a.fh + 1) * kr;
      r.apack = static_cast<uint64_t>(kTcBM) * r.p.K;
    }
  } else {
    // CI / WIN: channels on N on a CTA pair (each SM streams half the filter
    // tile) when the layer is long enough for >= 4 waves of 256-column pair
    // tiles (measured on B200: conv2 137 -> 125 us; the 13x13 layers, 1-2
    // ragged waves, run faster one CTA per tile); otherwise -- or with the
    // profiling knob LCNN_CONV_PAIR=0 -- the orientation with more useful
    // flops per operand byte
    static const int pair_knob = [] {
      const char* e = std::getenv("LCNN_CONV_PAIR");
      return e ? (e[0] == '0' ? 0 : 2) : 1;  // 0 off, 2 forced on, 1 by waves
    }();
    const uint64_t pair_tiles =
        (ncols + 2 * kTcBM - 1) / (2 * kTcBM) * ((a.co + co_tile_n(a.co) - 1) / co_tile_n(a.co));
    // ... and only when the channel tile keeps the MMA efficient: N = C_o
    // tile < 192 would sit on the ~96-cycle per-MMA floor (VGG conv1_2, C_o
    // = 64: N = 64 runs at a third of the tensor rate; channels on M with
    // 256-column tiles at half)
    const bool pair = pair_knob == 2 ||
                      (pair_knob == 1 && co_tile_n(a.co) >= 192 &&
                       pair_tiles >= 4ull * static_cast<uint64_t>(tc_sm_count() / 2));
    // TAPS (tap-sharing boxes) for layers whose channel planes are large
    // (H*W*N*4 >= 4 MB: activations far beyond L2, where the per-(tap,
    // channel-block) boxes are DRAM-latency-bound): measured on B200, VGG-16
    // conv1_2 / conv2_1 / conv2_2 3.9 / 1.05 / 1.9 ms -> 1.9 / 0.54 / 0.97 ms;
    // neutral at 56x56 and slower on AlexNet's 27x27 / 13x13 layers.
    // Profiling knob LCNN_CONV_TAPS: 0 off, 1 forced wherever supported.
    const bool big_planes = static_cast<uint64_t>(a.h) * a.w * a.n * 4 >= (4ull << 20);
    static const int taps_knob = [] {
      const char* e = std::getenv("LCNN_CONV_TAPS");
      return e ? (e[0] == '1' ? 2 : 0) : 1;
    }();
    if (r.p.g.mode == kModeCI && (taps_knob == 2 || (taps_knob == 1 && big_planes)) &&
        taps_geom(a).ok) {
      r.kind = kRouteTaps;
      r.p.g.mode = kModeTAPS;
      r.apack = static_cast<uint64_t>(a.co) * r.p.K;
      // C_o <= 64 at stride 1: row pairs fill the 128-row MMA (output rows
      // oh and oh + 1 on the two halves of M) instead of leaving half of it
      // padding.  Profiling knob LCNN_CONV_TAPS2=0 keeps one row per tile.
      static const bool taps2_off = [] {
        const char* e = std::getenv("LCNN_CONV_TAPS2");
        return e && e[0] == '0';
      }();
      if (!taps2_off && a.co <= 64 && a.stride == 1 && a.ho >= 2 &&
          a.precision == LCNN_PREC_TF32) {
        r.kind = kRouteTaps2;
        r.p.K = (a.fh + 1) * a.ci * a.fw;
        r.apack = static_cast<uint64_t>(kTcBM) * r.p.K;
      }
      return r;
    }
    // TAPS-N (tap-sharing boxes, channels on N, CTA pair) for 3x3 CI layers
    // whose planes are not TAPS-sized and whose rows fill 4-pixel blocks to
    // >= 87 %: measured on B200 (profiles/r01_conv_tapsn.txt), VGG-16 conv3_1
    // / conv3_2 / conv4_2 / conv5_1 310 / 582 / 566 / 187 -> 289 / 539 / 526 /
    // 179 us; slower on AlexNet's 5x5 conv2 (103 -> 125 us in the chain) and
    // its 13-wide layers (13 of 16 columns used).  Profiling knob LCNN_CONV_TAPSN: 0 off, 1 forced
    // wherever supported.
    static const int tapsn_knob = [] {
      const char* e = std::getenv("LCNN_CONV_TAPSN");
      return e ? (e[0] == '1' ? 2 : 0) : 1;
    }();
    const uint32_t owb4 = (a.wo + kTapsNPix - 1) / kTapsNPix * kTapsNPix;  // padded row
    const bool tapsn_fit = a.wo >= 14 && a.fw <= 3 && owb4 * 100 <= a.wo * 115 && !big_planes;
    if (r.p.g.mode == kModeCI && (tapsn_knob == 2 || (tapsn_knob == 1 && tapsn_fit)) &&
        tapsn_geom(a).ok) {
      r.kind = kRouteTapsN;
      r.p.g.mode = kModeTAPS;
      r.apack = static_cast<uint64_t>(a.co) * r.p.K;
      return r;
    }
    if (pair)
      r.kind = kRouteChwnPair;
    else
      r.kind = choose_co_on_n_traffic(a.co) ? kRouteChwnOnN : kRouteChwnOnM;
    r.apack = static_cast<uint64_t>(a.co) * r.p.K;
  }
  return r;
}

bool split_input(const ConvArgs& a, const ConvRoute& r) {
  return a.precision == LCNN_PREC_3XTF32 && r.kind != kRouteSimt && r.kind != kRouteNchwTc;
}

size_t packed_bytes(const ConvArgs& a, const ConvRoute& r) {
  // ROW images are sized for either orientation, so a bound computed without
  // the output extents (lcnn_conv_workspace_bytes) covers the route taken
  uint64_t floats = r.apack;
  if (r.kind == kRouteRowOnN || r.kind == kRouteRowOnM)
    floats = static_cast<uint64_t>(std::max(pack_rows(a.co, true), pack_rows(a.co, false))) * r.p.K;
  const uint64_t one = align_floats(floats);
  return (a.precision == LCNN_PREC_3XTF32 && r.kind != kRouteSimt ? 2 : 1) * one * 4;
}

size_t run_bytes(const ConvArgs& a, const ConvRoute& r) {
  const uint64_t nx = align_floats(static_cast<uint64_t>(a.n) * a.ci * a.h * a.w);
  const uint64_t ny = align_floats(static_cast<uint64_t>(a.n) * a.co * a.ho * a.wo);
  // [x_hi | x_lo] (3xTF32 split input), then for via-CHWN [x_chwn | y_chwn]
  return ((split_input(a, r) ? 2 * nx : 0) + (r.via_chwn ? nx + ny : 0)) * 4;
}

}  // namespace

size_t conv_packed_bytes(const ConvArgs& a) { return packed_bytes(a, route_conv(a)); }

size_t conv_workspace_bytes(const ConvArgs& a) {
  const ConvRoute r = route_conv(a);
  return packed_bytes(a, r) + run_bytes(a, r) + 512;
}

cudaError_t launch_conv_pack(const ConvArgs& a, void* packed, cudaStream_t s) {
  const ConvRoute r = route_conv(a);
  float* hi = static_cast<float*>(packed);
  float* lo = a.precision == LCNN_PREC_3XTF32 ? hi + packed_bytes(a, r) / 8 : nullptr;
  switch (r.kind) {
    case kRouteSimt:
      return cudaMemcpyAsync(hi, a.filters, r.apack * 4, cudaMemcpyDeviceToDevice, s);
    case kRouteNchwTc: {
      ConvGeomTc g{a.n, a.ci, a.h, a.w, a.co, a.fh, a.fw, a.stride, a.pad, a.ho, a.wo,
                   kModeNAT, 0, 0, 0};
      pack_filters_kernel<<<148 * 4, 256, 0, s>>>(a.filters, hi, nullptr, g, r.kp);
      break;
    }
    case kRouteRowOnN:
    case kRouteRowOnM:
      pack_filters_row_kernel<<<148 * 4, 256, 0, s>>>(
          a.filters, hi, lo, r.p.g, r.kind == kRouteRowOnN ? co_tile_n(a.co) : kTcBM, r.apack);
      break;
    case kRouteShare:
    case kRouteShareRes:
      pack_filters_row_kernel<<<148 * 4, 256, 0, s>>>(a.filters, hi, nullptr, r.p.g,
                                                      (a.co + 7) / 8 * 8, r.apack);
      break;
    case kRouteTaps2:
      pack_filters_taps2_kernel<<<148 * 4, 256, 0, s>>>(a.filters, hi, r.p.g, r.p.K);
      break;
    case kRouteRowPairs:
      pack_filters_row2_kernel<<<148 * 4, 256, 0, s>>>(a.filters, hi, r.p.g, r.apack);
      break;
    default:
      pack_filters_kernel<<<148 * 4, 256, 0, s>>>(a.filters, hi, lo, r.p.g, r.p.K);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_conv_packed(const ConvArgs& a, const void* packed, cudaStream_t s) {
  const ConvRoute r = route_conv(a);
  const float* w_hi = static_cast<const float*>(packed);
  const float* w_lo = a.precision == LCNN_PREC_3XTF32 ? w_hi + packed_bytes(a, r) / 8 : w_hi;
  if (r.kind == kRouteSimt) {
    ConvGeomSimt g{a.n, a.ci, a.h, a.w, a.co, a.fh, a.fw, a.stride, a.pad, a.ho, a.wo};
    const uint64_t total = static_cast<uint64_t>(a.n) * a.co * a.ho * a.wo;
    uint64_t blocks = (total + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    if (blocks == 0) blocks = 1;
    if (a.layout == LCNN_CHWN)
      lcnn_pdl::launch(conv_chwn_simt_kernel, static_cast<uint32_t>(blocks), 256, 0, s, a.src, w_hi, a.dst, g);
    else
      lcnn_pdl::launch(conv_nchw_simt_kernel, static_cast<uint32_t>(blocks), 256, 0, s, a.src, w_hi, a.dst, g);
    return cudaGetLastError();
  }
  if (r.kind == kRouteNchwTc) return launch_conv_nchw_tc(a, w_hi, r.kp, s);
  if (r.via_chwn) {
    // workspace: [inner run bytes | x_chwn | y_chwn]; NCHW [N][CHW] is the
    // transpose of CHWN [CHW][N]
    ConvArgs b = a;
    b.layout = LCNN_CHWN;
    ConvRoute inner = r;
    inner.via_chwn = false;
    uint8_t* ws = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(a.workspace) + 255) & ~uintptr_t(255));
    float* xc = reinterpret_cast<float*>(ws + run_bytes(b, inner));
    float* yc = xc + align_floats(static_cast<uint64_t>(a.n) * a.ci * a.h * a.w);
    cudaError_t e = launch_transpose2d(a.src, xc, a.n, static_cast<uint64_t>(a.ci) * a.h * a.w, s);
    if (e != cudaSuccess) return e;
    b.src = xc;
    b.dst = yc;
    b.workspace = ws;
    e = launch_conv_packed(b, packed, s);
    if (e != cudaSuccess) return e;
    return launch_transpose2d(yc, a.dst, static_cast<uint64_t>(a.co) * a.ho * a.wo, a.n, s);
  }
  const float* x_hi = a.src;
  const float* x_lo = a.src;
  if (split_input(a, r)) {
    const uint64_t nx = static_cast<uint64_t>(a.n) * a.ci * a.h * a.w;
    float* bh = reinterpret_cast<float*>(
        (reinterpret_cast<uintptr_t>(a.workspace) + 255) & ~uintptr_t(255));
    float* bl = bh + align_floats(nx);
    cudaError_t e = launch_split_hilo(a.src, bh, bl, nx, s);
    if (e != cudaSuccess) return e;
    x_hi = bh;
    x_lo = bl;
  }
  ConvTcArgs t{a, r.p, w_hi, w_lo, x_hi, x_lo};
  if (r.kind == kRouteShare || r.kind == kRouteShareRes)
    return launch_chwn_share(t, r.kind == kRouteShareRes, s);
  if (a.blk && (a.blk != LCNN_CONV_OUT_HWCN32 || r.kind != kRouteRowPairs))
    return cudaErrorNotSupported;  // blocked activations: row-pair producer only here
  if (r.kind == kRouteRowOnN) return launch_chwn_row<true>(t, s);
  if (r.kind == kRouteRowOnM) return launch_chwn_row<false>(t, s);
  if (r.kind == kRouteRowPairs) return launch_chwn_row<false>(t, s, true);
  if (r.kind == kRouteTaps) return taps_acc2_ok(a) ? launch_chwn_taps_acc2(t, s) : launch_chwn_taps(t, s);
  if (r.kind == kRouteTaps2) return launch_chwn_taps(t, s, true);
  if (r.kind == kRouteTapsN) return launch_chwn_tapsn(t, s);
  if (r.kind == kRouteChwnPair) return launch_chwn_tc<true, true>(t, s);
  return r.kind == kRouteChwnOnN ? launch_chwn_tc<true>(t, s) : launch_chwn_tc<false>(t, s);
}

// Convolution + max pooling fused (SharePoolOut): CHWN, TF32, a layer the
// SHARE route takes, pooling stride 2 with a 2- or 3-wide square window.
// profiling knob LCNN_TAPS_POOL=0: a TAPS row-pair conv and its 2x2 pool run as two kernels
bool taps_pool_knob() {
  static const bool on = [] {
    const char* e = std::getenv("LCNN_TAPS_POOL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Also a TAPS row-pair layer (C_o <= 64, e.g. VGG conv1_2) with a 2x2 window:
// the pool runs in the row-pair epilogue (TapsParams::pool).
bool conv_maxpool_fusable(const ConvArgs& a, uint32_t pwin, uint32_t pstride) {
  if (a.layout != LCNN_CHWN || a.precision != LCNN_PREC_TF32) return false;
  if (pstride != kPoolStride || (pwin != 2 && pwin != 3) || a.ho < pwin || a.wo < pwin)
    return false;
  const ConvRoute r = route_conv(a);
  if (r.via_chwn) return false;
  if (r.kind == kRouteTaps2) return pwin == 2 && taps_pool_knob();
  if (r.kind == kRouteTaps) return pwin == 2 && taps_pool_knob() && taps_acc2_ok(a);
  return r.kind == kRouteShare;
}

cudaError_t launch_conv_maxpool_packed(const ConvArgs& a, const void* packed, uint32_t pwin,
                                       uint32_t pstride, cudaStream_t s) {
  if (!conv_maxpool_fusable(a, pwin, pstride)) return cudaErrorInvalidValue;
  const ConvRoute r = route_conv(a);
  const float* w = static_cast<const float*>(packed);
  ConvTcArgs t{a, r.p, w, w, a.src, a.src};
  const uint32_t hp = (a.ho - pwin) / pstride + 1, wp = (a.wo - pwin) / pstride + 1;
  if (a.blk && (a.blk != LCNN_CONV_IN_HWCN32 || r.kind != kRouteTaps2))
    return cudaErrorNotSupported;  // blocked input: the TAPS row-pair consumer only
  if (r.kind == kRouteTaps2) return launch_chwn_taps(t, s, true, a.dst, hp, wp);
  if (r.kind == kRouteTaps) return launch_chwn_taps_acc2(t, s, a.dst, hp, wp);
  // profiling knob LCNN_SHAREPOOL_STORE=tma: staged TMA stores of the pooled
  // chunks (one ring slot fewer) instead of direct lane stores
  static const bool tma = [] {
    const char* e = std::getenv("LCNN_SHAREPOOL_STORE");
    return e && e[0] == 't';
  }();
  // (2-wide windows keep 4 open pool columns: 128 accumulator registers,
  // which the direct-store epilogue would spill -- they always stage)
  if (pwin == 2) return launch_chwn_share_pool<2, false>(t, a.dst, hp, wp, s);
  return tma ? launch_chwn_share_pool<3, false>(t, a.dst, hp, wp, s)
             : launch_chwn_share_pool<3, true>(t, a.dst, hp, wp, s);
}

bool conv_hwcn32_ok(const ConvArgs& a, uint32_t pwin, uint32_t pstride) {
  if (a.layout != LCNN_CHWN || a.precision != LCNN_PREC_TF32 || a.n % 128 || !a.blk) return false;
  const ConvRoute r = route_conv(a);
  if (a.blk == LCNN_CONV_OUT_HWCN32)  // ROW row pairs with the quad-box epilogue
    return pwin == 0 && r.kind == kRouteRowPairs && !r.via_chwn &&
           (uint64_t{a.wo} * a.n) % 128 == 0;
  if (a.blk == LCNN_CONV_IN_HWCN32)  // TAPS row pairs with the fused pool
    return pwin != 0 && conv_maxpool_fusable(a, pwin, pstride) && r.kind == kRouteTaps2;
  return false;
}

// One-shot form: pack into the front of the workspace, run with the rest.
cudaError_t launch_conv(const ConvArgs& a, cudaStream_t s) {
  const ConvRoute r = route_conv(a);
  uint8_t* ws = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(a.workspace) + 255) & ~uintptr_t(255));
  cudaError_t e = launch_conv_pack(a, ws, s);
  if (e != cudaSuccess) return e;
  ConvArgs b = a;
  b.workspace = ws + packed_bytes(a, r);
  return launch_conv_packed(b, ws, s);
}

}  // namespace lcnn_impl
