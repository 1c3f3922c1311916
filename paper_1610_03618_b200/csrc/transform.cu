// NCHW <-> CHWN layout transformation on sm_100a.
//
// Reference: /root/reference/proj/src/layout.cpp
//   transform_tiled  :99-120  flattens CHWN<->NCHW to a 2D transpose of the
//                             [C*H*W] x [N] view through a tile^2 scratch
//   transpose2d_tiled:31-68   the tile loop (scalar or 8-byte "wide" copies)
//   transform_naive  :77-97   4-loop permutation for any layout pair
// Paper: PAPER.md Fig. 7b (shared-memory tile + float2 when N >= 64).
//
// B200 design.  The op is pure data movement, so the roofline is HBM copy
// bandwidth: 2 x N*C*H*W*4 bytes per call (bench.cpp:202).  Each CTA moves a
// TR x TC tile:
//   * load phase: every warp reads 4 source rows x 128 B with 128-bit loads
//     (L1::no_allocate: the data is touched once);
//   * the tile lands in shared memory with a row pitch of TC+1 words, which
//     makes both the transposed scalar stores and the column reads
//     conflict-free (pitch == 1 mod 32 banks);
//   * store phase: every warp writes 4 destination rows x 128 B with 128-bit
//     streaming stores.
// When a row length is not a multiple of 4 floats (e.g. AlexNet's 3x227x227
// input, or odd batches) the affected side falls back to scalar 32-bit
// accesses, still one full 128-byte line per warp instruction.
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "internal.h"

namespace lcnn_dev {

template <int TR, int TC, bool VLD, bool VST>
__global__ void __launch_bounds__(kThreads)
    transpose2d_kernel(const float* __restrict__ src, float* __restrict__ dst,
                       uint32_t R, uint32_t C, uint32_t tiles_c) {
  LCNN_PDL_ENTRY();
  static_assert(TR % 32 == 0 && TC % 32 == 0, "tile edges are warp multiples");
  constexpr int P = TC + 1;  // shared-memory pitch, == 1 (mod 32)
  __shared__ float tile[TR * P];

  // batched form (blockIdx.y): independent R x C matrices back to back
  // (NCHW <-> NHWC is N transposes of C x HW)
  const uint64_t bofs = static_cast<uint64_t>(blockIdx.y) * R * C;
  src += bofs;
  dst += bofs;
  const uint32_t t = blockIdx.x;
  const uint32_t tr = t / tiles_c;
  const uint32_t tc = t - tr * tiles_c;
  const uint32_t r0 = tr * TR;
  const uint32_t c0 = tc * TC;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;

  // ---- load: src[r0 .. r0+TR) x [c0 .. c0+TC) -> tile[r][c] -------------
  if constexpr (VLD) {
    // warp slot = 4 rows x 8 float4 (128 B per row)
    constexpr int kSlotsC = TC / 32;          // float4 column groups of 8
    constexpr int kSlots = (TR / 4) * kSlotsC;
    float4 v[kSlots / kWarps];
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int c4 = (ws % kSlotsC) * 8 + (lane & 7);
      const int r = (ws / kSlotsC) * 4 + (lane >> 3);
      const uint32_t gr = r0 + r, gc = c0 + c4 * 4;
      v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < R && gc < C) {
        v[i] = ldg_stream(reinterpret_cast<const float4*>(
            src + static_cast<uint64_t>(gr) * C + gc));
      }
    }
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int c4 = (ws % kSlotsC) * 8 + (lane & 7);
      const int r = (ws / kSlotsC) * 4 + (lane >> 3);
      float* row = tile + r * P + c4 * 4;
      row[0] = v[i].x;
      row[1] = v[i].y;
      row[2] = v[i].z;
      row[3] = v[i].w;
    }
  } else {
    // warp slot = 1 row x 32 floats
    constexpr int kSlotsC = TC / 32;
    constexpr int kSlots = TR * kSlotsC;
    float v[kSlots / kWarps];
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int c = (ws % kSlotsC) * 32 + lane;
      const int r = ws / kSlotsC;
      const uint32_t gr = r0 + r, gc = c0 + c;
      v[i] = 0.f;
      if (gr < R && gc < C) v[i] = __ldg(src + static_cast<uint64_t>(gr) * C + gc);
    }
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int c = (ws % kSlotsC) * 32 + lane;
      const int r = ws / kSlotsC;
      tile[r * P + c] = v[i];
    }
  }
  __syncthreads();

  // ---- store: dst[c0 .. c0+TC) x [r0 .. r0+TR) <- tile[r][c] -------------
  if constexpr (VST) {
    // warp slot = 4 dst rows (source columns) x 8 float4 (128 B per row)
    constexpr int kSlotsR = TR / 32;
    constexpr int kSlots = (TC / 4) * kSlotsR;
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int r4 = (ws % kSlotsR) * 8 + (lane & 7);
      const int c = (ws / kSlotsR) * 4 + (lane >> 3);
      const uint32_t gr = r0 + r4 * 4, gc = c0 + c;
      if (gr < R && gc < C) {
        float4 o;
        o.x = tile[(r4 * 4 + 0) * P + c];
        o.y = tile[(r4 * 4 + 1) * P + c];
        o.z = tile[(r4 * 4 + 2) * P + c];
        o.w = tile[(r4 * 4 + 3) * P + c];
        stg_stream(reinterpret_cast<float4*>(dst + static_cast<uint64_t>(gc) * R + gr), o);
      }
    }
  } else {
    constexpr int kSlotsR = TR / 32;
    constexpr int kSlots = TC * kSlotsR;
#pragma unroll
    for (int i = 0; i < kSlots / kWarps; ++i) {
      const int ws = warp + i * kWarps;
      const int r = (ws % kSlotsR) * 32 + lane;
      const int c = ws / kSlotsR;
      const uint32_t gr = r0 + r, gc = c0 + c;
      if (gr < R && gc < C) {
        stg_stream(dst + static_cast<uint64_t>(gc) * R + gr, tile[r * P + c]);
      }
    }
  }
}

// Transpose with one short side (S = min(R, C) <= 16, the small batches of an
// N-sharded run: CHWN [CHW][N] with N = 256/G).  The 32-edge tiles above
// would be mostly empty (N = 8: 3/4 of every tile) with scalar side
// accesses.  Here a CTA owns a run of B = kSmallChunk / S long-side indices;
// both the read and the write of that run are S contiguous segments (or one
// contiguous block), moved with 128-bit accesses when aligned:
//   SMALL_C (C = S): src rows [l0, l0+B) are one block of B*S floats; dst
//                     holds S runs dst[c*R + l0 .. +B)
//   !SMALL_C (R = S): src holds S runs src[r*C + l0 .. +B); dst columns
//                     [l0, l0+B) are one block of B*S floats.
// Shared memory holds the run as [s][B + 1] (odd pitch for the transposed side).
constexpr int kSmallChunk = 4096;  // floats per CTA (16 KB in + 16 KB out)

template <int S, bool SMALL_C, bool VEC>
__global__ void __launch_bounds__(kThreads)
    transpose_small_kernel(const float* __restrict__ src, float* __restrict__ dst, uint32_t R,
                           uint32_t C) {
  LCNN_PDL_ENTRY();
  constexpr uint32_t B = (kSmallChunk / S) / 4 * 4;  // long-side indices per CTA
  constexpr uint32_t P = B + 1;                       // smem pitch (odd)
  __shared__ float sm[S * P];
  const uint32_t L = SMALL_C ? R : C;  // long side
  const uint32_t l0 = blockIdx.x * B;
  const uint32_t nb = min(B, L - l0);  // long-side indices in this run
  const uint32_t blk = nb * S;         // floats of the contiguous block
  // 1) the contiguous side -> smem[s][l]
  if constexpr (SMALL_C) {
    const float* blk_src = src + static_cast<uint64_t>(l0) * S;
    if constexpr (VEC) {
      constexpr uint32_t kIt = (B * S / 4 + kThreads - 1) / kThreads;
      float4 q[kIt];
#pragma unroll
      for (uint32_t it = 0; it < kIt; ++it) {
        const uint32_t i = threadIdx.x + it * kThreads;
        if (i < blk / 4) q[it] = ldg_stream(reinterpret_cast<const float4*>(blk_src) + i);
      }
#pragma unroll
      for (uint32_t it = 0; it < kIt; ++it) {
        const uint32_t i = threadIdx.x + it * kThreads;
        if (i < blk / 4) {
          const float e[4] = {q[it].x, q[it].y, q[it].z, q[it].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t f = 4 * i + j, l = f / S, c = f - l * S;
            sm[c * P + l] = e[j];
          }
        }
      }
    } else {
      for (uint32_t f = threadIdx.x; f < blk; f += kThreads) {
        const uint32_t l = f / S, c = f - l * S;
        sm[c * P + l] = __ldg(blk_src + f);
      }
    }
  } else {
    // S runs of nb floats each: src[r*C + l0 ..]
#pragma unroll
    for (uint32_t r = 0; r < S; ++r) {
      const float* run = src + static_cast<uint64_t>(r) * C + l0;
      if constexpr (VEC) {
        for (uint32_t i = threadIdx.x; i < nb / 4; i += kThreads) {
          const float4 q = ldg_stream(reinterpret_cast<const float4*>(run) + i);
          float* d = sm + r * P + 4 * i;
          d[0] = q.x; d[1] = q.y; d[2] = q.z; d[3] = q.w;
        }
      } else {
        for (uint32_t l = threadIdx.x; l < nb; l += kThreads) sm[r * P + l] = __ldg(run + l);
      }
    }
  }
  __syncthreads();
  // 2) smem -> the other side
  if constexpr (SMALL_C) {
    // S runs of nb floats: dst[c*R + l0 ..]
#pragma unroll
    for (uint32_t c = 0; c < S; ++c) {
      float* run = dst + static_cast<uint64_t>(c) * R + l0;
      if constexpr (VEC) {
        for (uint32_t i = threadIdx.x; i < nb / 4; i += kThreads) {
          const float* q = sm + c * P + 4 * i;
          stg_stream(reinterpret_cast<float4*>(run) + i, make_float4(q[0], q[1], q[2], q[3]));
        }
      } else {
        for (uint32_t l = threadIdx.x; l < nb; l += kThreads) stg_stream(run + l, sm[c * P + l]);
      }
    }
  } else {
    // one block: dst[(l0 + l)*S + r]
    float* blk_dst = dst + static_cast<uint64_t>(l0) * S;
    if constexpr (VEC) {
      for (uint32_t i = threadIdx.x; i < blk / 4; i += kThreads) {
        float e[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t f = 4 * i + j, l = f / S, r = f - l * S;
          e[j] = sm[r * P + l];
        }
        stg_stream(reinterpret_cast<float4*>(blk_dst) + i, make_float4(e[0], e[1], e[2], e[3]));
      }
    } else {
      for (uint32_t f = threadIdx.x; f < blk; f += kThreads) {
        const uint32_t l = f / S, r = f - l * S;
        stg_stream(blk_dst + f, sm[r * P + l]);
      }
    }
  }
}

// N = 1 (or any 1 x L) transpose: a copy.  A vectorised kernel rather than
// cudaMemcpyAsync: the D2D copy engine moved VGG's 12.8 MB activation at
// ~1.8 TB/s (transform_1 sweep, round 2).
// Each thread keeps kCopyUnroll 16-B loads in flight before its stores (one
// load per thread per trip left ~1.8 us of a 25 MB copy's ~5 us as latency).
constexpr int kCopyUnroll = 4;
__global__ void __launch_bounds__(kThreads)
    copy_f4_kernel(const float4* __restrict__ src, float4* __restrict__ dst, uint64_t n4) {
  LCNN_PDL_ENTRY();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x;
  for (; i + (kCopyUnroll - 1) * stride < n4; i += kCopyUnroll * stride) {
    float4 v[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) v[u] = ldg_stream(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) stg_stream(dst + i + u * stride, v[u]);
  }
  for (; i < n4; i += stride) stg_stream(dst + i, ldg_stream(src + i));
}

// Generic permutation between any two of the four layouts (layout.cpp:77-97
// semantics), as a batched 2-D problem.  Let a be the source's unit-stride
// logical dim and b the destination's, i and j the other two:
//   a != b : for every (i, j), dst[b-major] = transpose(src[a-major]) -- a
//            32 x 32 tile through shared memory (pitch 33), reads coalesced
//            along a, writes along b (NCHW<->NHWC, CHWN<->NHWC, ...);
//   a == b : both sides share the innermost dim (CHWN<->HWCN: runs of N):
//            contiguous runs copied with the outer three dims permuted (one
//            warp per run; runs shorter than 32 floats as a flat copy in
//            destination order).
// NCHW<->NHWC is N independent C x HW transposes: the tiled 128-bit
// transpose2d kernels above, batched over blockIdx.y (4.4 -> 6.8 TB/s at
// N = 128).  Round 1 ran one thread per destination element with a strided
// source gather (uncoalesced on one side).
struct PermGeom {
  uint32_t A, B;          // extents of a (src unit stride) and b (dst unit stride)
  uint32_t I, J;          // extents of the other two dims
  uint32_t tiles_a, tiles_b;
  FastDiv div_tiles_a, div_J;
  uint64_t sb, si, sj;    // source strides of b, i, j (a is 1)
  uint64_t da, di, dj;    // destination strides of a, i, j (b is 1)
};

__global__ void __launch_bounds__(kThreads)
    permute_tile_kernel(const float* __restrict__ src, float* __restrict__ dst, PermGeom g) {
  LCNN_PDL_ENTRY();
  __shared__ float tile[32][33];
  const uint32_t tiles = g.tiles_a * g.tiles_b;
  const uint64_t total = static_cast<uint64_t>(tiles) * g.I * g.J;
  for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
    const uint32_t ij = static_cast<uint32_t>(u / tiles);
    const uint32_t t = static_cast<uint32_t>(u - static_cast<uint64_t>(ij) * tiles);
    uint32_t tb, ta, i, j;
    g.div_tiles_a.divmod(t, tb, ta);
    g.div_J.divmod(ij, i, j);
    const uint32_t a0 = ta * 32, b0 = tb * 32;
    const uint64_t sbase = i * g.si + j * g.sj, dbase = i * g.di + j * g.dj;
    const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;  // 32 x 8 threads
    __syncthreads();  // the previous unit's readers are done with the tile
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const uint32_t a = a0 + lx, b = b0 + ly + r;
      if (a < g.A && b < g.B) tile[ly + r][lx] = __ldg(src + sbase + b * g.sb + a);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const uint32_t b = b0 + lx, a = a0 + ly + r;
      if (a < g.A && b < g.B) stg_stream(dst + dbase + a * g.da + b, tile[lx][ly + r]);
    }
  }
}

// a == b: runs of A contiguous floats; outer dims (b, i, j) permuted.
__global__ void __launch_bounds__(kThreads)
    permute_runs_kernel(const float* __restrict__ src, float* __restrict__ dst, PermGeom g) {
  LCNN_PDL_ENTRY();
  // one warp per run; B here is the third outer dim (i, j, b)
  const uint64_t runs = static_cast<uint64_t>(g.B) * g.I * g.J;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x) >> 5; w < runs;
       w += (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5) {
    const uint32_t ij = static_cast<uint32_t>(w / g.B);
    const uint32_t b = static_cast<uint32_t>(w - static_cast<uint64_t>(ij) * g.B);
    uint32_t i, j;
    g.div_J.divmod(ij, i, j);
    const float* s = src + b * g.sb + i * g.si + j * g.sj;
    float* d = dst + b * g.da + i * g.di + j * g.dj;
    for (uint32_t x = lane; x < g.A; x += 32) stg_stream(d + x, __ldg(s + x));
  }
}

// a == b, written in destination order: element e of the destination is
// x = e % A of run e / A, and the runs (b fastest, then j, then i) are
// contiguous in the destination -- so every warp stores 32 consecutive
// 16-byte (VEC) or 4-byte words, and reads runs of A floats (CHWN -> HWCN at
// N = 8: 32-byte runs, one sector each) instead of one warp per run.
template <int W>  // floats per word: 4 (16 B), 2 (8 B) or 1
__global__ void __launch_bounds__(kThreads)
    permute_runs_flat_kernel(const float* __restrict__ src, float* __restrict__ dst, PermGeom g,
                             FastDiv div_a, FastDiv div_b, uint64_t total) {
  LCNN_PDL_ENTRY();
  for (uint64_t e = (blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x); e < total;
       e += static_cast<uint64_t>(gridDim.x) * kThreads) {
    uint32_t run, x;
    div_a.divmod(static_cast<uint32_t>(e), run, x);  // total < 2^32 (host check)
    uint32_t ij, b, i, j;
    div_b.divmod(run, ij, b);
    g.div_J.divmod(ij, i, j);
    const float* sp = src + b * g.sb + i * g.si + j * g.sj + static_cast<uint64_t>(x) * W;
    if constexpr (W == 4) {
      stg_stream(reinterpret_cast<float4*>(dst) + e, ldg_stream(reinterpret_cast<const float4*>(sp)));
    } else if constexpr (W == 2) {
      reinterpret_cast<float2*>(dst)[e] = __ldg(reinterpret_cast<const float2*>(sp));
    } else {
      stg_stream(dst + e, __ldg(sp));
    }
  }
}

}  // namespace lcnn_dev

namespace lcnn_impl {

using namespace lcnn_dev;

namespace {

template <int TR, int TC>
cudaError_t launch_tile(const float* src, float* dst, uint32_t R, uint32_t C,
                        bool vld, bool vst, cudaStream_t s, uint32_t batch = 1) {
  const uint32_t tiles_r = (R + TR - 1) / TR;
  const uint32_t tiles_c = (C + TC - 1) / TC;
  const uint64_t tiles = static_cast<uint64_t>(tiles_r) * tiles_c;
  if (tiles > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<uint32_t>(tiles), batch);
  if (vld && vst)
    lcnn_pdl::launch(transpose2d_kernel<TR, TC, true, true>, grid, kThreads, 0, s, src, dst, R, C, tiles_c);
  else if (vld)
    lcnn_pdl::launch(transpose2d_kernel<TR, TC, true, false>, grid, kThreads, 0, s, src, dst, R, C, tiles_c);
  else if (vst)
    lcnn_pdl::launch(transpose2d_kernel<TR, TC, false, true>, grid, kThreads, 0, s, src, dst, R, C, tiles_c);
  else
    lcnn_pdl::launch(transpose2d_kernel<TR, TC, false, false>, grid, kThreads, 0, s, src, dst, R, C, tiles_c);
  return cudaGetLastError();
}

bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// `batch` R x C -> C x R transposes, both sides > 16 (the tiled kernels)
cudaError_t launch_transpose2d_tiled(const float* src, float* dst, uint32_t batch, uint32_t R,
                                     uint32_t C, cudaStream_t s) {
  // 128-bit accesses need every row start 16-byte aligned.
  const bool vld = (C % 4 == 0) && aligned16(src);
  const bool vst = (R % 4 == 0) && aligned16(dst);
  if (C >= 64) {
    if (R >= 64) return launch_tile<64, 64>(src, dst, R, C, vld, vst, s, batch);
    return launch_tile<32, 64>(src, dst, R, C, vld, vst, s, batch);
  }
  if (R >= 64) return launch_tile<64, 32>(src, dst, R, C, vld, vst, s, batch);
  return launch_tile<32, 32>(src, dst, R, C, vld, vst, s, batch);
}

}  // namespace

cudaError_t launch_transpose2d(const float* src, float* dst, uint64_t rows,
                               uint64_t cols, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const uint32_t R = static_cast<uint32_t>(rows);
  const uint32_t C = static_cast<uint32_t>(cols);
  // a 1 x L (or L x 1) transpose is a copy (N = 1 after sharding)
  if (R == 1 || C == 1) {
    const uint64_t n = rows * cols;
    if (n % 4 || !aligned16(src) || !aligned16(dst))
      return cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, s);
    uint64_t blocks = (n / 4 + kThreads * kCopyUnroll - 1) / (kThreads * kCopyUnroll);
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    lcnn_pdl::launch(copy_f4_kernel, static_cast<uint32_t>(blocks), kThreads, 0, s,
                     reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), n / 4);
    return cudaGetLastError();
  }
  const uint32_t S = R < C ? R : C;
  if (S <= 16) {
    const bool small_c = C <= R;
    const uint32_t L = small_c ? R : C;
    // 128-bit accesses: the block start l0*S and the run starts r*C / c*R
    // (with l0 a multiple of 4) are 16-byte aligned when L % 4 == 0
    const bool vec = aligned16(src) && aligned16(dst) && (L % 4 == 0);
    cudaError_t err = cudaErrorNotSupported;
    auto go = [&](auto s_tag) {
      constexpr int SS = decltype(s_tag)::value;
      constexpr uint32_t B = (kSmallChunk / SS) / 4 * 4;
      const uint32_t blocks = (L + B - 1) / B;
      if (small_c) {
        if (vec) lcnn_pdl::launch(transpose_small_kernel<SS, true, true>, blocks, kThreads, 0, s, src, dst, R, C);
        else lcnn_pdl::launch(transpose_small_kernel<SS, true, false>, blocks, kThreads, 0, s, src, dst, R, C);
      } else {
        if (vec) lcnn_pdl::launch(transpose_small_kernel<SS, false, true>, blocks, kThreads, 0, s, src, dst, R, C);
        else lcnn_pdl::launch(transpose_small_kernel<SS, false, false>, blocks, kThreads, 0, s, src, dst, R, C);
      }
      err = cudaGetLastError();
    };
    switch (S) {
#define LCNN_S(k) case k: go(std::integral_constant<int, k>{}); break;
      LCNN_S(2) LCNN_S(3) LCNN_S(4) LCNN_S(5) LCNN_S(6) LCNN_S(7) LCNN_S(8) LCNN_S(9)
      LCNN_S(10) LCNN_S(11) LCNN_S(12) LCNN_S(13) LCNN_S(14) LCNN_S(15) LCNN_S(16)
#undef LCNN_S
      default: break;
    }
    return err;
  }
  return launch_transpose2d_tiled(src, dst, 1, R, C, s);
}

cudaError_t launch_permute4d(const float* src, float* dst, uint32_t n,
                             uint32_t c, uint32_t h, uint32_t w, int src_layout,
                             int dst_layout, cudaStream_t s) {
  // logical extents, indexed n=0, c=1, h=2, w=3
  const uint32_t ext[4] = {n, c, h, w};
  // memory order (outermost..innermost) per layout code, tensor.hpp:16
  static const int order[4][4] = {{0, 1, 2, 3},   // NCHW
                                  {1, 2, 3, 0},   // CHWN
                                  {0, 2, 3, 1},   // NHWC
                                  {2, 3, 1, 0}};  // HWCN
  uint64_t ss[4], ds[4];  // source / destination stride of each logical dim
  uint64_t acc = 1;
  for (int k = 3; k >= 0; --k) {
    ss[order[src_layout][k]] = acc;
    acc *= ext[order[src_layout][k]];
  }
  acc = 1;
  for (int k = 3; k >= 0; --k) {
    ds[order[dst_layout][k]] = acc;
    acc *= ext[order[dst_layout][k]];
  }
  const uint64_t total = static_cast<uint64_t>(n) * c * h * w;
  if (total == 0) return cudaSuccess;
  // NCHW <-> NHWC: n independent (C x HW) <-> (HW x C) transposes -- the
  // tiled 128-bit transpose kernels, batched over n
  const uint64_t hw = static_cast<uint64_t>(h) * w;
  if (((src_layout == 0 && dst_layout == 2) ||
       (src_layout == 2 && dst_layout == 0)) &&
      c > 16 && hw > 16 && hw < (1ull << 31) && n <= 65535) {
    const bool fwd = src_layout == 0;  // NCHW (tensor.hpp:16 codes: NCHW 0, NHWC 2)
    return launch_transpose2d_tiled(src, dst, n, fwd ? c : static_cast<uint32_t>(hw),
                                    fwd ? static_cast<uint32_t>(hw) : c, s);
  }
  const int a = order[src_layout][3], b = order[dst_layout][3];
  int rest[3], nr = 0;
  for (int d = 0; d < 4; ++d)
    if (d != a && d != b) rest[nr++] = d;
  PermGeom g{};
  if (a != b) {
    g.A = ext[a];
    g.B = ext[b];
    g.I = ext[rest[0]];
    g.J = ext[rest[1]];
    g.sb = ss[b];
    g.si = ss[rest[0]];
    g.sj = ss[rest[1]];
    g.da = ds[a];
    g.di = ds[rest[0]];
    g.dj = ds[rest[1]];
    g.tiles_a = (g.A + 31) / 32;
    g.tiles_b = (g.B + 31) / 32;
    g.div_tiles_a = FastDiv(g.tiles_a);
    g.div_J = FastDiv(g.J);
    const uint64_t units = static_cast<uint64_t>(g.tiles_a) * g.tiles_b * g.I * g.J;
    const uint64_t blocks = units < 148ull * 32 ? units : 148ull * 32;
    lcnn_pdl::launch(permute_tile_kernel, static_cast<uint32_t>(blocks), kThreads, 0, s, src, dst, g);
    return cudaGetLastError();
  }
  // a == b: runs of ext[a]; the three outer dims are rest[0..2]
  g.A = ext[a];
  g.B = ext[rest[0]];
  g.I = ext[rest[1]];
  g.J = ext[rest[2]];
  g.sb = ss[rest[0]];
  g.si = ss[rest[1]];
  g.sj = ss[rest[2]];
  g.da = ds[rest[0]];
  g.di = ds[rest[1]];
  g.dj = ds[rest[2]];
  g.div_J = FastDiv(g.J);
  // short runs (A < 32 floats: a small N-shard of CHWN <-> HWCN): measured on
  // B200 at N = 8, 0.60 -> 4.5 TB/s; long runs keep one warp per run (N = 128:
  // 6.16 vs 6.01 TB/s flat)
  if (total < (1ull << 32) && ext[a] < 32) {
    // destination-ordered flat copy (runs of any length; 16-B words when the
    // runs, and so every run start, are 16-B aligned): the three outer dims
    // ordered by destination stride, b the fastest, then j, then i
    int r[3] = {rest[0], rest[1], rest[2]};
    for (int x = 0; x < 3; ++x)
      for (int y = x + 1; y < 3; ++y)
        if (ds[r[y]] < ds[r[x]]) std::swap(r[x], r[y]);
    g.B = ext[r[0]];
    g.J = ext[r[1]];
    g.I = ext[r[2]];
    g.sb = ss[r[0]];
    g.sj = ss[r[1]];
    g.si = ss[r[2]];
    g.div_J = FastDiv(g.J);
    const bool al16 = aligned16(src) && aligned16(dst);
    const bool al8 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7u) == 0;
    const int W = g.A % 4 == 0 && al16 ? 4 : (g.A % 2 == 0 && al8 ? 2 : 1);
    const uint32_t A = g.A / W;
    const uint64_t words = total / W;
    uint64_t blocks = (words + kThreads - 1) / kThreads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    const uint32_t nb = static_cast<uint32_t>(blocks);
    if (W == 4)
      lcnn_pdl::launch(permute_runs_flat_kernel<4>, nb, kThreads, 0, s, src, dst, g, FastDiv(A),
                       FastDiv(g.B), words);
    else if (W == 2)
      lcnn_pdl::launch(permute_runs_flat_kernel<2>, nb, kThreads, 0, s, src, dst, g, FastDiv(A),
                       FastDiv(g.B), words);
    else
      lcnn_pdl::launch(permute_runs_flat_kernel<1>, nb, kThreads, 0, s, src, dst, g, FastDiv(A),
                       FastDiv(g.B), words);
    return cudaGetLastError();
  }
  const uint64_t warps = static_cast<uint64_t>(g.B) * g.I * g.J;
  uint64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  lcnn_pdl::launch(permute_runs_kernel, static_cast<uint32_t>(blocks), kThreads, 0, s, src, dst, g);
  return cudaGetLastError();
}

}  // namespace lcnn_impl
