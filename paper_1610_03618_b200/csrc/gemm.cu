// Tensor-core (tcgen05, kind::tf32) GEMM on sm_100a, plus the fp32 SIMT
// path used when bit-level fp32 accuracy is requested.
//
// Reference: /root/reference/proj/src/conv.cpp:252-304 gemm_blocked (64^3
// blocks, fp32 partials flushed to fp64 every 16 k) and softmax.cpp:182-184
// fc_forward.  C (m x n) = A (m x k) * B (k x n), all row-major fp32.
//
// B200 design (one CTA per 128 x 128 output tile, warp-specialised):
//   warp 0      : TMA producer -- A tile 128(M) x 32(K) K-major and B tile
//                 32(K) x 128(N) MN-major (4 boxes of 32 N), SWIZZLE_128B,
//                 into a STAGES-deep shared-memory ring (mbarrier full/empty);
//   warp 1      : one elected thread issues tcgen05.mma.kind::tf32
//                 (M=128, N=128, K=8) x 4 per stage into a 128-column TMEM
//                 accumulator; tcgen05.commit frees the smem stage;
//   warps 2..5  : epilogue -- tcgen05.ld 32x32b.x32 TMEM -> registers ->
//                 global (each warp owns the 32 TMEM lanes of its quarter).
// Row-major B (N contiguous) is consumed as an MN-major operand directly, so
// neither operand is ever transposed or re-packed in HBM.
//
// Precision modes: TF32 (one MMA chain); 3xTF32 chains three operand sets
// hi*hi + hi*lo + lo*hi into the same accumulator (hi = x rounded to tf32,
// lo = tf32(x - hi), split by one elementwise kernel), giving ~fp32 accuracy.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <stdio.h>

#include "../../include/lcnn_cuda.h"
#include "common.cuh"
#include "internal.h"
#include "tc_gemm.cuh"

namespace lcnn_dev {

using namespace lcnn_tc;

// Plain GEMM operands: A (m x k) K-major, B (k x n) MN-major, both via 2D TMA
// (A box 32x128, B four boxes 32x32).  seg selects (A_hi,B_hi) (A_hi,B_lo)
// (A_lo,B_hi) in 3xTF32 mode; in TF32 mode only segment 0 exists.
struct GemmLoader {
  CUtensorMap a[2];
  CUtensorMap b[2];
  // grouped B (n % 32 == 0): one 3D box {32 n, 32 k, 8 groups} per stage over
  // the view {32, k, n/32} whose group stride (128 B) is smaller than the row
  // pitch -- it lands exactly as the 8 MN-major 32-column atoms, replacing 8
  // 2D boxes (TMA cost is mostly per box: scripts/tma_bench.cu)
  bool grouped;
  static constexpr bool kZeroSmem = false;
  static constexpr int kSteps = kTcBK / 8;
  static constexpr bool kResidentA = false;
  __device__ uint64_t desc_a(const uint8_t* sa, int k) const {
    return smem_desc_sw128(sa + k * 32, 16, 1024);
  }
  __device__ uint64_t desc_b(const uint8_t* sb, int k) const {
    return smem_desc_sw128(sb + k * 1024, 4096, 512, 1);
  }
  __device__ void prefetch() const {
    tma_prefetch(&a[0]);
    tma_prefetch(&b[0]);
  }
  __device__ uint32_t resident_bytes() const { return 0; }
  __device__ void load_resident(void*, uint64_t*) const {}
  __device__ uint32_t resident_offset(uint32_t) const { return 0; }
  struct State {
    uint32_t m0, n0;
  };
  __device__ State begin(uint32_t m0, uint32_t n0, uint32_t) const { return State{m0, n0}; }
  __device__ void load(State& st, uint32_t seg, uint32_t k, void* sa, void* sb,
                       uint64_t* bar) const {
    const CUtensorMap* am = &a[seg == 2 ? 1 : 0];
    const CUtensorMap* bm = &b[seg == 1 ? 1 : 0];
    tma_load_2d(sa, am, bar, k * kTcBK, st.m0);
    if (grouped) {
      tma_load_3d(sb, bm, bar, 0, k * kTcBK, st.n0 / 32);
    } else {
#pragma unroll
      for (int j = 0; j < kPBN / 32; ++j)
        tma_load_2d(static_cast<uint8_t*>(sb) + j * 4096, bm, bar, st.n0 + 32 * j, k * kTcBK);
    }
  }
};

template <bool kTma>
struct GemmOutT {
  float* c;
  uint64_t ldc;
  uint32_t M, N;
  // TMA-store epilogue (kTma; needs ldc % 4 == 0 and a 16-B aligned C): 2D
  // view {N, M}, box {32, 32}, SWIZZLE_128B -- the stream-K fragments of the
  // skinny fc GEMMs become TMA add-reductions instead of per-lane vector atomics
  CUtensorMap y;
  static constexpr bool kTmaStore = kTma, kTmaTransposed = false;
  __device__ __forceinline__ void tma_chunk(const void* box, uint32_t m0, uint32_t n0,
                                            bool add) const {
    if (n0 >= N || m0 >= M) return;
    if (add)
      tma_add_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
    else
      tma_store_2d(&y, box, static_cast<int32_t>(n0), static_cast<int32_t>(m0));
  }
  __device__ __forceinline__ void store32(uint32_t m, uint32_t n0, const float* v,
                                          bool add) const {
    if (n0 >= N) return;  // warp-uniform
    if (n0 + 32 <= N && ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(c) & 15u) == 0) {
      warp_store_rows32(m < M ? c + m * ldc + n0 : nullptr, v, add);
    } else if (m < M) {
      store_row32(c + m * ldc + n0, n0, N, v, add);
    }
  }
};


// fc layer on pre-packed weights (softmax.cpp:182-184 fc_forward with the
// weights of a network layer, constant across forwards).  B = W^T packed once
// K-major [n][k] (one 2D TMA box {32 k, 256 n} per stage, SWIZZLE_128B -- W
// is row-major [k][n], and N = 1000-style widths would otherwise need eight
// 32-column boxes per stage).  A = the activations, either K-major rows
// [m][k] (an NCHW producer's flatten) or MN-major [k][m] (kAMn: a CHWN
// producer -- the image index is contiguous, so the flatten the reference
// performs before fc (net.cpp:258-262) becomes the operand load itself and
// the transposing transform is skipped).
template <bool kAMn>
struct FcLoader {
  CUtensorMap a[2];
  const float* bimg[2];  // packed weights hi / lo: swizzled stage images [nt][kb][256][32]
  uint32_t kbn;          // k-blocks
  uint32_t bn;           // weight rows (output columns) one stage loads: 256, or 128
  uint32_t pf_ahead;     // k-blocks of weights prefetched into L2 ahead of the TMA loads
  bool a_grouped;  // MN-major A, m % 128 == 0: one 3D box {32, 32 k, 4 groups}
  bool skip_a;     // profiling (LCNN_TC_PROBE bit 4): no activation loads
  // the next fc layer's packed weights (nullptr: none): each CTA prefetches
  // its 1/grid share into L2 after issuing its last load, so the next layer
  // starts on L2 hits while this one drains
  const uint8_t* next_w;
  uint64_t next_bytes;
  static constexpr bool kTailPrefetch = true;
  static constexpr bool kZeroSmem = false;
  static constexpr bool kResidentA = false;
  static constexpr int kSteps = kTcBK / 8;
  __device__ void tail_prefetch(uint32_t cta, uint32_t grid) const {
    if (!next_w) return;
    const uint64_t share = (next_bytes / grid + 255) / 256 * 256;
    const uint64_t lo = share * cta;
    if (lo >= next_bytes) return;
    uint64_t len = next_bytes - lo < share ? next_bytes - lo : share;
    for (uint64_t off = 0; off < len; off += (1u << 20)) {
      const uint64_t b = len - off < (1u << 20) ? len - off : (1u << 20);
      bulk_prefetch_l2(next_w + lo + off, static_cast<uint32_t>(b) & ~15u);
    }
  }
  __device__ uint64_t desc_a(const uint8_t* sa, int k) const {
    return kAMn ? smem_desc_sw128(sa + k * 1024, 4096, 512, 1) : smem_desc_sw128(sa + k * 32, 16, 1024);
  }
  __device__ uint64_t desc_b(const uint8_t* sb, int k) const {
    return smem_desc_sw128(sb + k * 32, 16, 1024);
  }
  __device__ void prefetch() const { tma_prefetch(&a[0]); }
  __device__ uint32_t resident_bytes() const { return 0; }
  __device__ void load_resident(void*, uint64_t*) const {}
  __device__ uint32_t resident_offset(uint32_t) const { return 0; }
  struct State {
    uint32_t m0, n0;
  };
  __device__ State begin(uint32_t m0, uint32_t n0, uint32_t) const { return State{m0, n0}; }
  __device__ void load(State& st, uint32_t seg, uint32_t k, void* sa, void* sb,
                       uint64_t* bar) const {
    const CUtensorMap* am = &a[seg == 2 ? 1 : 0];
    const int32_t k0 = static_cast<int32_t>(k * kTcBK);
    if (skip_a) {
    } else if constexpr (kAMn) {
      if (a_grouped) {
        tma_load_3d(sa, am, bar, 0, k0, static_cast<int32_t>(st.m0 / 32));
      } else {
#pragma unroll
        for (int j = 0; j < kTcBM / 32; ++j)
          tma_load_2d(static_cast<uint8_t*>(sa) + j * 4096, am, bar,
                      static_cast<int32_t>(st.m0 + 32 * j), k0);
      }
    } else {
      tma_load_2d(sa, am, bar, k0, static_cast<int32_t>(st.m0));
    }
    // a 128-row half of a 256-row image tile keeps its swizzle phase (128 % 8 == 0)
    const float* w = bimg[seg == 1 ? 1 : 0] +
                     ((static_cast<uint64_t>(st.n0 / kPBN) * kbn + k) * kPBN + st.n0 % kPBN) * kTcBK;
    bulk_load(sb, w, bn * kTcBK * 4, bar);
    // the weight stage kPrefetch k-blocks ahead goes to L2 now
    if (pf_ahead && k + pf_ahead < kbn)
      bulk_prefetch_l2(w + static_cast<uint64_t>(pf_ahead) * kPBN * kTcBK, bn * kTcBK * 4);
  }
};

// The K-major SWIZZLE_128B stage images of W^T: img[((t * KB + kb) * 256 +
// r) * 32 + (c ^ (r & 7)) * 4 + e] = W[k = kb*32 + 4c + e][n = t*256 + r]
// (zero past k / n).  One thread per (n, 4-k chunk) group of the image; W is
// read through a 32 x 33 shared tile so both sides stay coalesced.
__global__ void __launch_bounds__(256)
    pack_fc_kernel(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo,
                   uint32_t K, uint32_t N) {
  __shared__ float t[32][33];
  const uint32_t KB = (K + 31) / 32, NT = (N + kPBN - 1) / kPBN;
  const uint32_t nblk = NT * (kPBN / 32);  // 32-row blocks of n
  const uint32_t tiles = nblk * KB;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t kb = tile % KB, nb = tile / KB;
    const uint32_t k0 = kb * 32, n0 = nb * 32;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
      const uint32_t r = i / 32, c = i % 32;  // r: k, c: n (coalesced along n)
      t[r][c] = (k0 + r < K && n0 + c < N) ? w[static_cast<uint64_t>(k0 + r) * N + n0 + c] : 0.0f;
    }
    __syncthreads();
    const uint32_t nt = n0 / kPBN, rbase = n0 % kPBN;
    float* base_hi = hi + (static_cast<uint64_t>(nt) * KB + kb) * kPBN * 32;
    float* base_lo = lo ? lo + (static_cast<uint64_t>(nt) * KB + kb) * kPBN * 32 : nullptr;
    for (uint32_t i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
      const uint32_t rr = i / 32, slot = i % 32;  // image row (n) and float slot (coalesced)
      const uint32_t r = rbase + rr;
      const uint32_t kk = ((slot >> 2) ^ (r & 7)) * 4 + (slot & 3);
      const float v = t[kk][rr];
      const uint64_t o = static_cast<uint64_t>(r) * 32 + slot;
      if (base_lo) {
        uint32_t u;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
        const float h = __uint_as_float(u);
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v - h));
        base_hi[o] = h;
        base_lo[o] = __uint_as_float(u);
      } else {
        base_hi[o] = v;
      }
    }
  }
}

// Zero a 2D region of 32-bit words (stream-K output regions, the softmax
// non-finite flag): a PDL kernel, so it does not break the layer chain the
// way a cudaMemset node would.
__global__ void __launch_bounds__(256)
    zero2d_kernel(uint32_t* __restrict__ p, uint64_t pitch, uint64_t width, uint64_t total) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint64_t r = i / width;
    p[r * pitch + (i - r * width)] = 0u;
  }
}

// 3xTF32 operand split: hi = x rounded to tf32 (low 13 mantissa bits zero,
// so the tensor core consumes it exactly), lo = tf32(x - hi).
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void split_hilo_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                  float* __restrict__ lo, uint64_t count) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i];
    const float h = to_tf32(v);
    hi[i] = h;
    lo[i] = to_tf32(v - h);
  }
}

// fp32 CUDA-core GEMM (64x64 tile, 4x4 per thread) with the reference's
// accumulation split (conv.cpp:252-293): fp32 products and 16-deep fp32
// partial sums, flushed into an fp64 running total -- for LCNN_PREC_FP32 and
// shapes TMA cannot describe.
__global__ void __launch_bounds__(256)
    gemm_fp32_simt_kernel(const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ c, uint64_t M, uint64_t N, uint64_t K) {
  LCNN_PDL_ENTRY();
  __shared__ float sa[16][64 + 4];
  __shared__ float sb[16][64 + 4];
  const uint64_t m0 = blockIdx.y * 64ull, n0 = blockIdx.x * 64ull;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double master[4][4] = {};
  for (uint64_t k0 = 0; k0 < K; k0 += 16) {
    float acc[4][4] = {};
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i % 16, mm = i / 16;
      sa[kk][mm] = (m0 + mm < M && k0 + kk < K) ? a[(m0 + mm) * K + k0 + kk] : 0.0f;
      const int nn = i % 64, kb = i / 64;
      sb[kb][nn] = (n0 + nn < N && k0 + kb < K) ? b[(k0 + kb) * N + n0 + nn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = sa[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sb[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) master[i][j] += acc[i][j];
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) c[m * N + n] = static_cast<float>(master[i][j]);
    }
}

}  // namespace lcnn_dev

namespace lcnn_impl {

using namespace lcnn_dev;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

}  // namespace

// 2D fp32 tensor map: dims {inner, outer}, row pitch in bytes, box {bi, bo}.
// swizzle: 0 = SWIZZLE_128B (K-major operands), 1 = SWIZZLE_128B_ATOM_32B
// (MN-major 32-bit operands), 2 = none (interleaved core-matrix images)
bool make_tmap_2d(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer,
                  uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer, bool mn_major) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

bool make_tmap(CUtensorMap* m, const float* base, uint32_t rank, const uint64_t* dims,
               const uint64_t* pitches_bytes, const uint32_t* box, const uint32_t* estrides,
               int swizzle) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (uint32_t i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = estrides ? estrides[i] : 1;
    if (i + 1 < rank) s[i] = pitches_bytes[i];
  }
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), d, s, b, e,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle == 1   ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
             : swizzle == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE
                            : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Launch the persistent kernel with a TMA-store epilogue when C allows it.
template <class Loader>
cudaError_t launch_gemm_out(const Loader& L, float* c, uint64_t ldc, uint32_t m, uint32_t n,
                            const Sched& sc, cudaStream_t s) {
  if (ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(c) & 15u) == 0) {
    lcnn_dev::GemmOutT<true> O{c, ldc, m, n};
    const uint64_t dims[2] = {n, m};
    const uint64_t pitch[1] = {ldc * 4};
    const uint32_t box[2] = {32, 32};
    Sched se = sc;
    sched_epi(se, se.ctl_off - se.resident_off > 16 ? se.ctl_off - se.resident_off : 0);
    if (se.smem_bytes <= kMaxDynSmem && make_tmap(&O.y, c, 2, dims, pitch, box, nullptr, 0))
      return launch_persistent(L, O, se, s);
  }
  lcnn_dev::GemmOutT<false> O{c, ldc, m, n};
  return launch_persistent(L, O, sc, s);
}

bool tc_gemm_supported(uint64_t m, uint64_t n, uint64_t k, const void* a, const void* b) {
  // TMA: 16-byte aligned bases and row pitches
  return m > 0 && n > 0 && k > 0 && (k % 4 == 0) && (n % 4 == 0) &&
         ((reinterpret_cast<uintptr_t>(a) & 15u) == 0) &&
         ((reinterpret_cast<uintptr_t>(b) & 15u) == 0) && m < (1ull << 31) && n < (1ull << 31) &&
         k < (1ull << 31);
}

cudaError_t launch_zero2d(void* p, uint64_t pitch_words, uint64_t width_words, uint64_t rows,
                          cudaStream_t s) {
  const uint64_t total = width_words * rows;
  if (!total) return cudaSuccess;
#ifdef LCNN_PROFILING_KNOBS
  // LCNN_SKIP_ZERO=1: no stream-K zeroing launches (wrong sums; timing only)
  static const bool skip = [] {
    const char* e = std::getenv("LCNN_SKIP_ZERO");
    return e && e[0] == '1';
  }();
  if (skip && pitch_words > 1) return cudaSuccess;
#endif
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  return lcnn_pdl::launch(zero2d_kernel, static_cast<uint32_t>(blocks), 256, 0, s,
                          static_cast<uint32_t*>(p), pitch_words, width_words, total);
}

cudaError_t launch_split_hilo(const float* x, float* hi, float* lo, uint64_t count,
                              cudaStream_t s) {
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  lcnn_pdl::launch(split_hilo_kernel, static_cast<uint32_t>(blocks ? blocks : 1), 256, 0, s, x, hi, lo, count);
  return cudaGetLastError();
}

size_t gemm_workspace_bytes(uint64_t m, uint64_t n, uint64_t k, int precision) {
  if (precision != LCNN_PREC_3XTF32) return 0;
  return (2 * m * k + 2 * k * n) * sizeof(float) + 64;
}

// precision TF32: a, b used directly.  3XTF32: ws holds a_hi, a_lo, b_hi, b_lo.
cudaError_t launch_gemm_tc(const float* a, const float* b, float* c, uint64_t m, uint64_t n,
                           uint64_t k, int precision, void* ws, cudaStream_t s) {
  GemmLoader L;
  const float *a0 = a, *a1 = a, *b0 = b, *b1 = b;
  if (precision == LCNN_PREC_3XTF32) {
    float* w = static_cast<float*>(ws);
    float* ahi = w;
    float* alo = ahi + m * k;
    float* bhi = alo + m * k;
    float* blo = bhi + k * n;
    cudaError_t e = launch_split_hilo(a, ahi, alo, m * k, s);
    if (e == cudaSuccess) e = launch_split_hilo(b, bhi, blo, k * n, s);
    if (e != cudaSuccess) return e;
    a0 = ahi; a1 = alo; b0 = bhi; b1 = blo;
  }
  if (!make_tmap_2d(&L.a[0], a0, k, m, k * 4, kTcBK, kTcBM, false) ||
      !make_tmap_2d(&L.a[1], a1, k, m, k * 4, kTcBK, kTcBM, false))
    return cudaErrorInvalidValue;
  L.grouped = n % 32 == 0;
  if (L.grouped) {
    const uint64_t dims[3] = {32, k, n / 32};
    const uint64_t pitch[2] = {n * 4, 128};
    const uint32_t box[3] = {32, kTcBK, kPBN / 32};
    if (!make_tmap(&L.b[0], b0, 3, dims, pitch, box, nullptr, 1) ||
        !make_tmap(&L.b[1], b1, 3, dims, pitch, box, nullptr, 1))
      return cudaErrorInvalidValue;
  } else if (!make_tmap_2d(&L.b[0], b0, n, k, n * 4, 32, kTcBK, true) ||
             !make_tmap_2d(&L.b[1], b1, n, k, n * 4, 32, kTcBK, true)) {
    return cudaErrorInvalidValue;
  }
  Sched sc = make_sched(static_cast<uint32_t>((m + kTcBM - 1) / kTcBM),
                        static_cast<uint32_t>((n + kPBN - 1) / kPBN),
                        static_cast<uint32_t>((k + kTcBK - 1) / kTcBK),
                        precision == LCNN_PREC_3XTF32 ? 3 : 1, kPBN, false, true);
  const uint32_t zc = sched_zero_col(sc, kPBN);
  if (zc < n) {
    cudaError_t e = launch_zero2d(c + zc, n, n - zc, m, s);
    if (e != cudaSuccess) return e;
  }
  return launch_gemm_out(L, c, n, static_cast<uint32_t>(m), static_cast<uint32_t>(n), sc, s);
}

cudaError_t launch_gemm_fp32(const float* a, const float* b, float* c, uint64_t m, uint64_t n,
                             uint64_t k, cudaStream_t s) {
  const dim3 grid(static_cast<uint32_t>((n + 63) / 64), static_cast<uint32_t>((m + 63) / 64));
  lcnn_pdl::launch(gemm_fp32_simt_kernel, grid, 256, 0, s, a, b, c, m, n, k);
  return cudaGetLastError();
}

// Packed fc weights: [hi | lo (3xTF32 only)], each n x k floats, 256-B aligned.
size_t fc_packed_bytes(uint64_t k, uint64_t n, int precision) {
  const uint64_t one = ((n + kPBN - 1) / kPBN) * kPBN * ((k + 31) / 32) * 32 * sizeof(float);
  return (precision == LCNN_PREC_3XTF32 ? 2 : 1) * one;
}

size_t fc_workspace_bytes(uint64_t m, uint64_t k, int precision) {
  return precision == LCNN_PREC_3XTF32 ? 2 * ((m * k + 63) / 64 * 64) * sizeof(float) + 256 : 0;
}

cudaError_t launch_fc_pack(const float* w, uint64_t k, uint64_t n, int precision, void* packed,
                           cudaStream_t s) {
  float* hi = static_cast<float*>(packed);
  float* lo = precision == LCNN_PREC_3XTF32 ? hi + fc_packed_bytes(k, n, precision) / 8 : nullptr;
  const uint64_t tiles = ((n + kPBN - 1) / kPBN) * (kPBN / 32) * ((k + 31) / 32);
  const uint32_t grid = static_cast<uint32_t>(tiles < 148 * 8 ? tiles : 148 * 8);
  pack_fc_kernel<<<grid, 256, 0, s>>>(w, hi, lo, static_cast<uint32_t>(k), static_cast<uint32_t>(n));
  return cudaGetLastError();
}


namespace {

// Skinny fc GEMMs (m = one batch) are pure stream-K; fragments as short as 4
// k-blocks keep every SM streaming weights (fc8: 128 CTAs instead of 64).
constexpr uint32_t kFcMinSkIters = 4;

template <bool kAMn>
cudaError_t launch_fc_tc(const float* x, const void* packed, float* c, uint64_t m, uint64_t n,
                         uint64_t k, int precision, void* ws, cudaStream_t s,
                         unsigned long long* zsync, const void* next_packed, uint64_t next_bytes) {
  FcLoader<kAMn> L;
  L.next_w = static_cast<const uint8_t*>(next_packed);
  L.next_bytes = next_packed ? next_bytes : 0;
  const float* b0 = static_cast<const float*>(packed);
  const float* b1 = precision == LCNN_PREC_3XTF32 ? b0 + fc_packed_bytes(k, n, precision) / 8 : b0;
  const float *a0 = x, *a1 = x;
  if (precision == LCNN_PREC_3XTF32) {
    float* ah = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    float* al = ah + (m * k + 63) / 64 * 64;
    cudaError_t e = launch_split_hilo(x, ah, al, m * k, s);
    if (e != cudaSuccess) return e;
    a0 = ah;
    a1 = al;
  }
  L.bimg[0] = b0;
  L.bimg[1] = b1;
  L.kbn = static_cast<uint32_t>((k + kTcBK - 1) / kTcBK);
  L.bn = kPBN;
  static const uint32_t pf = [] {
    const char* e = std::getenv("LCNN_FC_PREFETCH");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  L.pf_ahead = pf;  // measured: L2 prefetch ahead of the ring only slows fc (0 = off)
  L.a_grouped = false;
  L.skip_a = false;
  if constexpr (kAMn) {
    L.a_grouped = m % kTcBM == 0;
    if (L.a_grouped) {
      const uint64_t dims[3] = {32, k, m / 32};
      const uint64_t pitch[2] = {m * 4, 128};
      const uint32_t box[3] = {32, kTcBK, kTcBM / 32};
      if (!make_tmap(&L.a[0], a0, 3, dims, pitch, box, nullptr, 1) ||
          !make_tmap(&L.a[1], a1, 3, dims, pitch, box, nullptr, 1))
        return cudaErrorInvalidValue;
    } else if (!make_tmap_2d(&L.a[0], a0, m, k, m * 4, 32, kTcBK, true) ||
               !make_tmap_2d(&L.a[1], a1, m, k, m * 4, 32, kTcBK, true)) {
      return cudaErrorInvalidValue;
    }
  } else if (!make_tmap_2d(&L.a[0], a0, k, m, k * 4, kTcBK, kTcBM, false) ||
             !make_tmap_2d(&L.a[1], a1, k, m, k * 4, kTcBK, kTcBM, false)) {
    return cudaErrorInvalidValue;
  }
  const uint32_t mt = static_cast<uint32_t>((m + kTcBM - 1) / kTcBM);
  const uint32_t segs = precision == LCNN_PREC_3XTF32 ? 3 : 1;
  {
    // cluster split-K when stream-K would leave each CTA fewer than 8
    // k-iterations (fc8: 4 -- its fragment reductions then outweigh the
    // loads; measured fc8 13.3 -> 10.8 us, while fc6 / fc7 at 31 / 14
    // iterations per CTA stay faster on stream-K over all 148 SMs): the
    // column tile (256 or 128) and split S <= 8 that put the most CTAs to
    // work, each CTA keeping >= 4 k-iterations (ties: the wider tile)
    const uint32_t sms = static_cast<uint32_t>(tc_sm_count()), iters = L.kbn * segs;
    const uint64_t sk_total = static_cast<uint64_t>(mt) * ((n + kPBN - 1) / kPBN) * iters;
    uint32_t best_bn = 0, best_s = 1, best_ctas = 0;
    // clusters of up to 16 CTAs (non-portable size) when the profiling knob
    // LCNN_FC_S16=1 asks for them
    static const uint32_t s_cap = [] {
      const char* e = std::getenv("LCNN_FC_S16");
      return (e && e[0] == '1') ? 16u : 8u;
    }();
    for (uint32_t bn : {static_cast<uint32_t>(kPBN), 128u}) {
      const uint32_t tiles = mt * static_cast<uint32_t>((n + bn - 1) / bn);
      uint32_t S = tiles ? sms / tiles : 0;
      S = std::min({S, s_cap, iters / 4});
      if (S >= 2 && tiles * S > best_ctas) {
        best_ctas = tiles * S;
        best_bn = bn;
        best_s = S;
      }
    }
    static const int splitk = [] {
      const char* e = std::getenv("LCNN_FC_SPLITK");
      // profiling knob: 0 = always stream-K, 2 = cluster split-K whenever it fits
      return e ? (e[0] == '0' ? 0 : (e[0] == '2' ? 2 : 1)) : 1;
    }();
    if (best_s >= 2 && splitk && (sk_total < 8ull * sms || splitk == 2)) {
      L.bn = best_bn;
      SplitK sk{};
      sk.mt = mt;
      sk.nt = static_cast<uint32_t>((n + best_bn - 1) / best_bn);
      sk.kbn = L.kbn;
      sk.iters = iters;
      sk.S = best_s;
      sk.bn = best_bn;
      sk.idesc = idesc_tf32(kTcBM, best_bn, kAMn, false);
      sk.a_bytes = kTcABytes;
      sk.stage_bytes = kTcABytes + best_bn * kTcBK * 4;
      sk.stage_stride = (sk.stage_bytes + 1023) / 1024 * 1024;
      sk.stages = 0;
      const uint32_t frag = kTcBM * kSplitPitch * 4;  // the parked fragment lives in the ring
      for (uint32_t st = kPStagesMax; st >= 2 && !sk.stages; --st) {
        const uint32_t ring = std::max(st * sk.stage_stride, (frag + 1023) / 1024 * 1024);
        if (1024 + ring + 16 + sizeof(PCtl) <= kMaxDynSmem) {
          sk.stages = st;
          sk.ctl_off = ring;
        }
      }
      sk.smem_bytes = 1024 + sk.ctl_off + static_cast<uint32_t>(sizeof(PCtl));
      sk.M = static_cast<uint32_t>(m);
      sk.N = static_cast<uint32_t>(n);
      const uint32_t probe = tc_probe_knob();
      sk.probe = probe;
      return launch_splitk(L, c, sk, s);
    }
  }
  Sched sc = make_sched(mt, static_cast<uint32_t>((n + kPBN - 1) / kPBN),
                        static_cast<uint32_t>((k + kTcBK - 1) / kTcBK), segs, kPBN, kAMn, false,
                        kFcMinSkIters);
  L.skip_a = (sc.probe & 4) != 0;
  if (L.skip_a) sc.stage_bytes -= sc.a_bytes;
  const uint32_t zc = sched_zero_col(sc, kPBN);
  if (zc < n) {
    cudaError_t e = sched_zero_region(sc, zsync, c + zc, n, n - zc, m, (zc / kPBN) * sc.mt,
                                      [s](float* p, uint64_t pitch, uint64_t width, uint64_t rows) {
                                        return launch_zero2d(p, pitch, width, rows, s);
                                      });
    if (e != cudaSuccess) return e;
  }
  return launch_gemm_out(L, c, n, static_cast<uint32_t>(m), static_cast<uint32_t>(n), sc, s);
}

}  // namespace

bool fc_tc_supported(uint64_t m, uint64_t n, uint64_t k, bool a_mn) {
  return m > 0 && n > 0 && k > 0 && k % 4 == 0 && (!a_mn || m % 4 == 0) && m < (1ull << 31) &&
         n < (1ull << 31) && k < (1ull << 31);
}

cudaError_t launch_fc_packed(const float* x, bool a_mn, const void* packed, float* c, uint64_t m,
                             uint64_t n, uint64_t k, int precision, void* ws, cudaStream_t s,
                             unsigned long long* zsync, const void* next_packed,
                             uint64_t next_bytes) {
  return a_mn ? launch_fc_tc<true>(x, packed, c, m, n, k, precision, ws, s, zsync, next_packed,
                                   next_bytes)
              : launch_fc_tc<false>(x, packed, c, m, n, k, precision, ws, s, zsync, next_packed,
                                    next_bytes);
}

}  // namespace lcnn_impl

extern "C" {

size_t lcnn_gemm_workspace_bytes(uint64_t m, uint64_t n, uint64_t k, int precision) {
  return lcnn_impl::gemm_workspace_bytes(m, n, k, precision);
}

}  // extern "C"
