// Max / average pooling in CHWN and NCHW on sm_100a.
//
// Reference: /root/reference/proj/src/pool.cpp
//   pool_plain CHWN   :98-134   lane buffer over the contiguous batch
//   pool_plain NCHW   :135-163  window loop per output
//   pool_coarsened    :178-270  fh x fw outputs per task, union staged once
//   pool_oracle       :49-84    fp64 ground truth, NCHW out
// Paper: PAPER.md Sec. 5 (coalescing along the fastest dimension; register
// coarsening of overlapped windows, auto-tuned factors).
//
// Bit-exactness contract (checked against the CPU reference by memcmp):
//   max : acc = (acc < v) ? v : acc, acc from -inf, taps in (y,x) order;
//   avg : fp32 adds from 0.0f in (y,x) order (no FMA contraction), then CHWN
//         multiplies by 1.0f/(wh*ww) (pool.cpp:104,129,261) while NCHW
//         divides by float(wh*ww) (pool.cpp:158).
// Register coarsening never changes a single output's tap order: union rows
// are visited top to bottom and each row left to right, so every output sees
// its own window in (y,x) order.
//
// CHWN kernel: lanes run along N with 128-bit loads (4 images per thread), so
// one warp instruction reads 512 contiguous bytes of a tap; each thread owns
// an FH x FW block of outputs and loads the receptive-field union of that
// block exactly once (UH x UW float4 loads for FH*FW outputs).
// NCHW kernel: a CTA stages a contiguous band of input rows of one (n,c)
// plane in shared memory (row-major, so the global read is one contiguous
// span), then threads compute FW consecutive outputs each from shared memory
// and write contiguous output rows.
#include <float.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace lcnn_dev {

struct ChwnGeom {
  const float* src;
  float* dst;
  uint32_t N, H, W, Ho, Wo;
  uint32_t nbh, nbw;   // output blocks along h and w
  FastDiv div_nv, div_nbw, div_nbh;
  uint32_t total;      // threads = C * nbh * nbw * NV
  float inv;           // 1.0f / (wh*ww) (average only)
  uint32_t wh, ww, s;  // runtime window (generic kernel only)
};

template <int VEC>
__device__ __forceinline__ typename Vec<VEC>::T load_tap(const float* p) {
  if constexpr (VEC == 4) {
    return __ldg(reinterpret_cast<const float4*>(p));
  } else {
    return __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void store_out(float* p, typename Vec<VEC>::T v) {
  if constexpr (VEC == 4) {
    stg_stream(reinterpret_cast<float4*>(p), v);
  } else {
    stg_stream(p, v);
  }
}

template <int WH, int WW, int S, int FH, int FW, int VEC, bool AVG>
__global__ void __launch_bounds__(kThreads)
    pool_chwn_kernel(ChwnGeom g) {
  LCNN_PDL_ENTRY();
  using T = typename Vec<VEC>::T;
  constexpr int UH = S * (FH - 1) + WH;
  constexpr int UW = S * (FW - 1) + WW;
  const uint32_t gid = blockIdx.x * kThreads + threadIdx.x;
  if (gid >= g.total) return;
  uint32_t item, nv, t, bw, bh, c;
  g.div_nv.divmod(gid, item, nv);
  g.div_nbw.divmod(item, t, bw);
  g.div_nbh.divmod(t, c, bh);
  const uint32_t oh0 = bh * FH, ow0 = bw * FW;
  const uint32_t ih0 = oh0 * S, iw0 = ow0 * S;
  const uint64_t N = g.N;
  const float* base =
      g.src + ((static_cast<uint64_t>(c) * g.H + ih0) * g.W + iw0) * N + nv * VEC;

  T acc[FH][FW];
#pragma unroll
  for (int by = 0; by < FH; ++by)
#pragma unroll
    for (int bx = 0; bx < FW; ++bx) acc[by][bx] = splat<VEC>(AVG ? 0.0f : -INFINITY);

#pragma unroll
  for (int y = 0; y < UH; ++y) {
    if (ih0 + y >= g.H) break;  // rows that only feed absent outputs
    T v[UW];
#pragma unroll
    for (int x = 0; x < UW; ++x) {
      v[x] = splat<VEC>(AVG ? 0.0f : -INFINITY);
      if (iw0 + x < g.W) v[x] = load_tap<VEC>(base + (static_cast<uint64_t>(y) * g.W + x) * N);
    }
#pragma unroll
    for (int by = 0; by < FH; ++by) {
      const int dy = y - by * S;
      if (dy < 0 || dy >= WH) continue;  // resolved at compile time
#pragma unroll
      for (int bx = 0; bx < FW; ++bx) {
#pragma unroll
        for (int xx = 0; xx < WW; ++xx) {
          if constexpr (AVG) {
            acc[by][bx] = add_tap(acc[by][bx], v[bx * S + xx]);
          } else {
            acc[by][bx] = max_tap(acc[by][bx], v[bx * S + xx]);
          }
        }
      }
    }
  }

  float* obase = g.dst + ((static_cast<uint64_t>(c) * g.Ho + oh0) * g.Wo + ow0) * N + nv * VEC;
#pragma unroll
  for (int by = 0; by < FH; ++by) {
#pragma unroll
    for (int bx = 0; bx < FW; ++bx) {
      if (oh0 + by < g.Ho && ow0 + bx < g.Wo) {
        T o = acc[by][bx];
        if constexpr (AVG) o = scale_out(o, g.inv);
        store_out<VEC>(obase + (static_cast<uint64_t>(by) * g.Wo + bx) * N, o);
      }
    }
  }
}

// Any window / stride, one output per thread (plain semantics).
template <int VEC, bool AVG>
__global__ void __launch_bounds__(kThreads) pool_chwn_generic_kernel(ChwnGeom g) {
  LCNN_PDL_ENTRY();
  using T = typename Vec<VEC>::T;
  const uint32_t gid = blockIdx.x * kThreads + threadIdx.x;
  if (gid >= g.total) return;
  uint32_t item, nv, t, ow, oh, c;
  g.div_nv.divmod(gid, item, nv);
  g.div_nbw.divmod(item, t, ow);
  g.div_nbh.divmod(t, c, oh);
  const uint64_t N = g.N;
  const float* base =
      g.src + ((static_cast<uint64_t>(c) * g.H + oh * g.s) * g.W + ow * g.s) * N + nv * VEC;
  T acc = splat<VEC>(AVG ? 0.0f : -INFINITY);
  for (uint32_t y = 0; y < g.wh; ++y) {
    for (uint32_t x = 0; x < g.ww; ++x) {
      const T v = load_tap<VEC>(base + (static_cast<uint64_t>(y) * g.W + x) * N);
      if constexpr (AVG) acc = add_tap(acc, v); else acc = max_tap(acc, v);
    }
  }
  if constexpr (AVG) acc = scale_out(acc, g.inv);
  store_out<VEC>(g.dst + ((static_cast<uint64_t>(c) * g.Ho + oh) * g.Wo + ow) * N + nv * VEC, acc);
}

// ---------------------------------------------------------------- NCHW ----
struct NchwGeom {
  const float* src;
  float* dst;
  uint32_t H, W, Ho, Wo;
  uint32_t band;       // output rows per CTA
  uint32_t nbands;     // bands per plane
  uint32_t nbw;        // output column blocks (of FW) per row
  FastDiv div_nbw;
  float divisor;       // float(wh*ww) (average only)
  uint32_t wh, ww, s;  // runtime window (generic kernel only)
};

// Stage `count` contiguous floats of global memory into shared memory.  The
// span is placed at smem offset (gp/4 mod 4) so that every 16-byte global
// vector lands on a 16-byte shared slot (conflict-free 128-bit stores); the
// caller indexes the staged span from the returned offset.
__device__ __forceinline__ uint32_t stage_span(float* sm, const float* gp, uint32_t count) {
  const uint32_t mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(gp) >> 2) & 3u);
  uint32_t head = (4u - mis) & 3u;
  if (head > count) head = count;
  if (threadIdx.x < head) sm[mis + threadIdx.x] = __ldg(gp + threadIdx.x);
  const uint32_t nvec = (count - head) >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(gp + head);
  float4* s4 = reinterpret_cast<float4*>(sm + mis + head);  // mis+head is 0 or 4
  uint32_t i = threadIdx.x;
  for (; i + 3 * kThreads < nvec; i += 4 * kThreads) {
    const float4 a = ldg_stream(g4 + i);
    const float4 b = ldg_stream(g4 + i + kThreads);
    const float4 c = ldg_stream(g4 + i + 2 * kThreads);
    const float4 d = ldg_stream(g4 + i + 3 * kThreads);
    s4[i] = a;
    s4[i + kThreads] = b;
    s4[i + 2 * kThreads] = c;
    s4[i + 3 * kThreads] = d;
  }
  for (; i < nvec; i += kThreads) s4[i] = ldg_stream(g4 + i);
  const uint32_t done = head + 4 * nvec;
  if (threadIdx.x < count - done) sm[mis + done + threadIdx.x] = __ldg(gp + done + threadIdx.x);
  return mis;
}

// Coarsening runs vertically first: a thread owns FH outputs of one column
// block, so lanes still walk consecutive output columns (stride-S shared
// reads) while the union rows shared by vertically adjacent windows are read
// once.  FW > 1 widens the block horizontally (more bank conflicts; offered
// for the auto-tuner to measure).
template <int WH, int WW, int S, int FH, int FW, bool AVG>
__global__ void __launch_bounds__(kThreads) pool_nchw_kernel(NchwGeom g) {
  LCNN_PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int UH = S * (FH - 1) + WH;
  constexpr int UW = S * (FW - 1) + WW;
  const uint32_t plane = blockIdx.x / g.nbands;
  const uint32_t b = blockIdx.x - plane * g.nbands;
  const uint32_t oh_begin = b * g.band;
  const uint32_t oh_cnt = min(g.band, g.Ho - oh_begin);
  const uint32_t ih_begin = oh_begin * S;
  const uint32_t ih_cnt = min(g.H - ih_begin, (oh_cnt - 1) * S + WH);
  const uint64_t hw = static_cast<uint64_t>(g.H) * g.W;
  const uint32_t off =
      stage_span(sm, g.src + plane * hw + static_cast<uint64_t>(ih_begin) * g.W, ih_cnt * g.W);
  __syncthreads();

  float* obase = g.dst + plane * static_cast<uint64_t>(g.Ho) * g.Wo +
                 static_cast<uint64_t>(oh_begin) * g.Wo;
  const uint32_t nrb = (oh_cnt + FH - 1) / FH;
  const uint32_t items = nrb * g.nbw;
  for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
    uint32_t rb, bw;
    g.div_nbw.divmod(it, rb, bw);
    const uint32_t r0 = rb * FH, ow0 = bw * FW;
    const float* win = sm + off + (r0 * S) * g.W + ow0 * S;
    float acc[FH][FW];
#pragma unroll
    for (int by = 0; by < FH; ++by)
#pragma unroll
      for (int bx = 0; bx < FW; ++bx) acc[by][bx] = AVG ? 0.0f : -INFINITY;
#pragma unroll
    for (int y = 0; y < UH; ++y) {
      if (r0 * S + y >= ih_cnt) break;  // rows that only feed absent outputs
      float v[UW];
#pragma unroll
      for (int x = 0; x < UW; ++x) {
        v[x] = (FW == 1 || ow0 * S + x < g.W) ? win[y * g.W + x] : 0.0f;
      }
#pragma unroll
      for (int by = 0; by < FH; ++by) {
        const int dy = y - by * S;
        if (dy < 0 || dy >= WH) continue;  // resolved at compile time
#pragma unroll
        for (int bx = 0; bx < FW; ++bx)
#pragma unroll
          for (int xx = 0; xx < WW; ++xx) {
            if constexpr (AVG) acc[by][bx] = add_tap(acc[by][bx], v[bx * S + xx]);
            else acc[by][bx] = max_tap(acc[by][bx], v[bx * S + xx]);
          }
      }
    }
#pragma unroll
    for (int by = 0; by < FH; ++by) {
      if (r0 + by >= oh_cnt) break;
      float* orow = obase + static_cast<uint64_t>(r0 + by) * g.Wo + ow0;
#pragma unroll
      for (int bx = 0; bx < FW; ++bx) {
        if (ow0 + bx < g.Wo) {
          const float o = AVG ? divide_out(acc[by][bx], g.divisor) : acc[by][bx];
          stg_stream(orow + bx, o);
        }
      }
    }
  }
}

// Persistent, pipelined NCHW kernel (strides 1 and 2, vertical coarsening).
// A work unit is either a group of whole (n,c) planes (small maps) or one
// band of output rows of a large plane; either way one contiguous input
// span.  One thread streams the spans of the next units into a g.pipe-deep
// shared-memory ring with TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx), so HBM reads of unit i+2 overlap the arithmetic of unit i.
// Spans are copied 16-byte aligned; the issuing thread patches the <= 3
// trailing floats a 16-byte granule cannot cover into the slot with plain
// loads (visible to the consumers through the barriers that separate issue
// from use), so the tap loop reads shared memory unconditionally.
constexpr int kPipeMax = 8;

struct NchwPipeGeom {
  const float* src;
  float* dst;
  uint32_t H, W, Ho, Wo;
  uint32_t planes;    // N*C
  uint32_t per_cta;   // planes per unit (whole-plane mode) or 1 (band mode)
  uint32_t band;      // output rows per unit (== Ho in whole-plane mode)
  uint32_t nbands;    // bands per plane (1 in whole-plane mode)
  uint32_t units;
  uint32_t stage_floats;  // ring slot size (multiple of 4)
  uint32_t pipe;          // ring slots (<= kPipeMax)
  FastDiv div_wo, div_plane_items;
  float divisor;
};

struct PipeUnit {
  uint32_t plane0, np, oh_begin, oh_cnt, ih_rows;
  const float* span;
  uint32_t count;
};

__device__ __forceinline__ PipeUnit pipe_unit(const NchwPipeGeom& g, uint32_t u, uint32_t S,
                                              uint32_t WH) {
  PipeUnit pu;
  if (g.nbands == 1) {
    pu.plane0 = u * g.per_cta;
    pu.np = min(g.per_cta, g.planes - pu.plane0);
    pu.oh_begin = 0;
    pu.oh_cnt = g.Ho;
    pu.ih_rows = pu.np * g.H;
  } else {
    pu.plane0 = u / g.nbands;
    pu.np = 1;
    pu.oh_begin = (u - pu.plane0 * g.nbands) * g.band;
    pu.oh_cnt = min(g.band, g.Ho - pu.oh_begin);
    pu.ih_rows = min(g.H - pu.oh_begin * S, (pu.oh_cnt - 1) * S + WH);
  }
  pu.span = g.src + static_cast<uint64_t>(pu.plane0) * g.H * g.W +
            static_cast<uint64_t>(pu.oh_begin) * S * g.W;
  pu.count = pu.ih_rows * g.W;
  return pu;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

template <int WH, int S, int FH, int FW, bool AVG>
__global__ void __launch_bounds__(kThreads) pool_nchw_pipe_kernel(NchwPipeGeom g) {
  LCNN_PDL_ENTRY();
  extern __shared__ __align__(16) float ring[];
  __shared__ __align__(8) uint64_t bar[kPipeMax];
  __shared__ uint32_t meta[kPipeMax][2];  // (float offset of the span, floats copied)
  constexpr int WW = WH;
  constexpr int UH = S * (FH - 1) + WH;
  constexpr int UW = S * (FW - 1) + WW;  // columns of one FW-wide output block's window union
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < g.pipe; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&bar[k]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](uint32_t i) {  // unit index i of this CTA -> ring slot i % g.pipe
    const uint32_t u = blockIdx.x + i * gridDim.x;
    if (u >= g.units) return;
    const PipeUnit pu = pipe_unit(g, u, S, WH);
    const uintptr_t addr = reinterpret_cast<uintptr_t>(pu.span);
    const uint32_t mis = static_cast<uint32_t>((addr >> 2) & 3u);
    const uint32_t bytes = ((mis + pu.count) * 4u) & ~15u;
    const uint32_t k = i % g.pipe;
    meta[k][0] = mis;
    meta[k][1] = bytes / 4;
    float* slot = ring + static_cast<size_t>(k) * g.stage_floats;
    for (uint32_t e = bytes / 4 > mis ? bytes / 4 - mis : 0; e < pu.count; ++e)
      slot[mis + e] = __ldg(pu.span + e);
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[k]));
    if (bytes) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                   : "memory");
      bulk_g2s(ring + static_cast<size_t>(k) * g.stage_floats,
               reinterpret_cast<const void*>(addr & ~uintptr_t(15)), bytes, &bar[k]);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
    }
  };

  if (threadIdx.x == 0)
    for (uint32_t i = 0; i + 1 < g.pipe; ++i) issue(i);

  for (uint32_t i = 0;; ++i) {
    const uint32_t u = blockIdx.x + i * gridDim.x;
    if (u >= g.units) break;
    if (threadIdx.x == 0) issue(i + g.pipe - 1);
    const uint32_t k = i % g.pipe;
    {
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[k]));
      const uint32_t parity = (i / g.pipe) & 1;
      asm volatile(
          "{\n.reg .pred p;\nWAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra WAIT_%=;\n}\n" ::"r"(b),
          "r"(parity)
          : "memory");
    }
    const PipeUnit pu = pipe_unit(g, u, S, WH);
    const float* sbuf = ring + static_cast<size_t>(k) * g.stage_floats + meta[k][0];
    const uint32_t nrb = (pu.oh_cnt + FH - 1) / FH;
    const uint32_t owc = (g.Wo + FW - 1) / FW;  // FW-wide output column blocks per row
    const uint32_t items = pu.np * nrb * owc;
    for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
      uint32_t p, rest, rb, oc;
      if (pu.np == 1) {
        p = 0;
        rest = it;
      } else {
        g.div_plane_items.divmod(it, p, rest);
      }
      g.div_wo.divmod(rest, rb, oc);  // div_wo divides by owc
      const uint32_t ow = oc * FW;
      const uint32_t r0 = rb * FH;
      const uint32_t prow = p * g.H;
      // an output (by, bx) takes its taps in (y, x) order from the shared
      // union rows / columns, the same order as an uncoarsened output
      float acc[FH][FW];
#pragma unroll
      for (int by = 0; by < FH; ++by)
#pragma unroll
        for (int bx = 0; bx < FW; ++bx) acc[by][bx] = AVG ? 0.0f : -INFINITY;
#pragma unroll
      for (int y = 0; y < UH; ++y) {
        const uint32_t rr = r0 * S + y;
        if (pu.np == 1 ? rr >= pu.ih_rows : rr >= g.H) break;  // rows of absent outputs
        const uint32_t e0 = (prow + rr) * g.W + ow * S;
        float v[UW];
#pragma unroll
        for (int x = 0; x < UW; ++x) {
          v[x] = sbuf[e0 + x];  // past the row end only for absent outputs (never stored)
        }
#pragma unroll
        for (int by = 0; by < FH; ++by) {
          const int dy = y - by * S;
          if (dy < 0 || dy >= WH) continue;
#pragma unroll
          for (int bx = 0; bx < FW; ++bx)
#pragma unroll
            for (int x = 0; x < WW; ++x) {
              if constexpr (AVG) acc[by][bx] = add_tap(acc[by][bx], v[bx * S + x]);
              else acc[by][bx] = max_tap(acc[by][bx], v[bx * S + x]);
            }
        }
      }
      float* orow = g.dst + static_cast<uint64_t>(pu.plane0 + p) * g.Ho * g.Wo +
                    static_cast<uint64_t>(pu.oh_begin + r0) * g.Wo + ow;
#pragma unroll
      for (int by = 0; by < FH; ++by) {
        if (r0 + by >= pu.oh_cnt) break;
#pragma unroll
        for (int bx = 0; bx < FW; ++bx) {
          if (ow + bx >= g.Wo) break;
          const float o = AVG ? divide_out(acc[by][bx], g.divisor) : acc[by][bx];
          stg_stream(orow + static_cast<uint64_t>(by) * g.Wo + bx, o);
        }
      }
    }
    __syncthreads();  // slot k is refilled by the issue() of iteration i + 1
  }
}

// Runtime window, staged the same way, one output per thread.
template <bool AVG>
__global__ void __launch_bounds__(kThreads) pool_nchw_generic_kernel(NchwGeom g) {
  LCNN_PDL_ENTRY();
  extern __shared__ float sm[];
  const uint32_t plane = blockIdx.x / g.nbands;
  const uint32_t b = blockIdx.x - plane * g.nbands;
  const uint32_t oh_begin = b * g.band;
  const uint32_t oh_cnt = min(g.band, g.Ho - oh_begin);
  const uint32_t ih_begin = oh_begin * g.s;
  const uint32_t ih_cnt = min(g.H - ih_begin, (oh_cnt - 1) * g.s + g.wh);
  const uint64_t hw = static_cast<uint64_t>(g.H) * g.W;
  const uint32_t off =
      stage_span(sm, g.src + plane * hw + static_cast<uint64_t>(ih_begin) * g.W, ih_cnt * g.W);
  __syncthreads();
  float* obase = g.dst + plane * static_cast<uint64_t>(g.Ho) * g.Wo +
                 static_cast<uint64_t>(oh_begin) * g.Wo;
  const uint32_t items = oh_cnt * g.Wo;
  for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
    uint32_t r, ow;
    g.div_nbw.divmod(it, r, ow);
    const float* win = sm + off + (r * g.s) * g.W + ow * g.s;
    float acc = AVG ? 0.0f : -INFINITY;
    for (uint32_t y = 0; y < g.wh; ++y)
      for (uint32_t x = 0; x < g.ww; ++x) {
        const float v = win[y * g.W + x];
        if constexpr (AVG) acc = add_tap(acc, v); else acc = max_tap(acc, v);
      }
    stg_stream(obase + static_cast<uint64_t>(r) * g.Wo + ow, AVG ? divide_out(acc, g.divisor) : acc);
  }
}

// Unstaged NCHW fallback for rows too wide to stage (W*wh*4 > smem budget).
template <bool AVG>
__global__ void __launch_bounds__(kThreads)
    pool_nchw_direct_kernel(const float* __restrict__ src, float* __restrict__ dst,
                            uint64_t total, uint32_t H, uint32_t W, uint32_t Ho,
                            uint32_t Wo, uint32_t wh, uint32_t ww, uint32_t s,
                            float divisor) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint64_t ow = i % Wo;
    const uint64_t t = i / Wo;
    const uint64_t oh = t % Ho;
    const uint64_t plane = t / Ho;
    const float* win = src + (plane * H + oh * s) * W + ow * s;
    float acc = AVG ? 0.0f : -INFINITY;
    for (uint32_t y = 0; y < wh; ++y)
      for (uint32_t x = 0; x < ww; ++x) {
        const float v = __ldg(win + static_cast<uint64_t>(y) * W + x);
        if constexpr (AVG) acc = add_tap(acc, v); else acc = max_tap(acc, v);
      }
    dst[i] = AVG ? divide_out(acc, divisor) : acc;
  }
}

// fp64 oracle (pool.cpp:49-84): any layout in via strides, NCHW out.
__global__ void pool_oracle_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                   uint32_t N, uint32_t C, uint32_t Ho, uint32_t Wo,
                                   uint64_t sn, uint64_t sc, uint64_t sh, uint64_t sw,
                                   uint32_t wh, uint32_t ww, uint32_t s, bool avg) {
  const uint64_t total = static_cast<uint64_t>(N) * C * Ho * Wo;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t ow = i % Wo;
    uint64_t t = i / Wo;
    const uint64_t oh = t % Ho;
    t /= Ho;
    const uint64_t c = t % C;
    const uint64_t n = t / C;
    const uint64_t base = n * sn + c * sc;
    double sum = 0.0;
    float best = src[base + oh * s * sh + ow * s * sw];
    for (uint32_t y = 0; y < wh; ++y)
      for (uint32_t x = 0; x < ww; ++x) {
        const float v = src[base + (oh * s + y) * sh + (ow * s + x) * sw];
        sum += v;
        best = max_tap(best, v);
      }
    dst[i] = avg ? static_cast<float>(sum / wh / ww) : best;
  }
}

}  // namespace lcnn_dev

namespace lcnn_impl {

using namespace lcnn_dev;

namespace {

constexpr uint32_t kStageBudget = 24 * 1024;  // bytes of input rows per CTA

inline uint32_t cdiv(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

template <int WH, int WW, int S, int FH, int FW, int VEC>
cudaError_t chwn_launch(const ChwnGeom& g, bool avg, cudaStream_t st) {
  const uint32_t blocks = cdiv(g.total, kThreads);
  if (avg) lcnn_pdl::launch(pool_chwn_kernel<WH, WW, S, FH, FW, VEC, true>, blocks, kThreads, 0, st, g);
  else lcnn_pdl::launch(pool_chwn_kernel<WH, WW, S, FH, FW, VEC, false>, blocks, kThreads, 0, st, g);
  return cudaGetLastError();
}

template <int WH, int WW, int S, int VEC>
bool chwn_dispatch_f(uint32_t fh, uint32_t fw, const ChwnGeom& g, bool avg,
                     cudaStream_t st, cudaError_t* err) {
#define LCNN_F(FH_, FW_)                                               \
  if (fh == FH_ && fw == FW_) {                                        \
    *err = chwn_launch<WH, WW, S, FH_, FW_, VEC>(g, avg, st);          \
    return true;                                                       \
  }
  LCNN_F(1, 1) LCNN_F(1, 2) LCNN_F(1, 3) LCNN_F(1, 4)
  LCNN_F(2, 1) LCNN_F(2, 2) LCNN_F(2, 3) LCNN_F(2, 4)
  LCNN_F(3, 1) LCNN_F(3, 2) LCNN_F(3, 3) LCNN_F(3, 4)
  LCNN_F(4, 1) LCNN_F(4, 2) LCNN_F(4, 3) LCNN_F(4, 4)
#undef LCNN_F
  return false;
}

template <int VEC>
bool chwn_dispatch(const PoolArgs& a, const ChwnGeom& g, cudaStream_t st, cudaError_t* err) {
  if (a.win_h == 2 && a.win_w == 2 && a.stride == 2)
    return chwn_dispatch_f<2, 2, 2, VEC>(a.fh, a.fw, g, a.avg, st, err);
  if (a.win_h == 3 && a.win_w == 3 && a.stride == 2)
    return chwn_dispatch_f<3, 3, 2, VEC>(a.fh, a.fw, g, a.avg, st, err);
  if (a.win_h == 3 && a.win_w == 3 && a.stride == 1)
    return chwn_dispatch_f<3, 3, 1, VEC>(a.fh, a.fw, g, a.avg, st, err);
  return false;
}

}  // namespace

cudaError_t launch_pool_chwn(const PoolArgs& a, cudaStream_t st) {
  const bool vec = (a.n % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.src) & 15u) == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.dst) & 15u) == 0);
  const uint32_t VEC = vec ? 4 : 1;
  ChwnGeom g;
  g.src = a.src;
  g.dst = a.dst;
  g.N = a.n;
  g.H = a.h;
  g.W = a.w;
  g.Ho = a.ho;
  g.Wo = a.wo;
  g.inv = 1.0f / static_cast<float>(a.win_h * a.win_w);  // pool.cpp:104
  g.wh = a.win_h;
  g.ww = a.win_w;
  g.s = a.stride;
  const uint32_t nv = a.n / VEC;
  g.div_nv = FastDiv(nv);

  cudaError_t err = cudaSuccess;
  // register-coarsened specialisations
  g.nbh = cdiv(a.ho, a.fh);
  g.nbw = cdiv(a.wo, a.fw);
  g.div_nbw = FastDiv(g.nbw);
  g.div_nbh = FastDiv(g.nbh);
  g.total = a.c * g.nbh * g.nbw * nv;
  if (g.total == 0) return cudaSuccess;
  if (vec ? chwn_dispatch<4>(a, g, st, &err) : chwn_dispatch<1>(a, g, st, &err)) return err;

  // generic: one output per thread, runtime window (same output bits)
  g.nbh = a.ho;
  g.nbw = a.wo;
  g.div_nbw = FastDiv(g.nbw);
  g.div_nbh = FastDiv(g.nbh);
  g.total = a.c * a.ho * a.wo * nv;
  const uint32_t blocks = cdiv(g.total, kThreads);
  if (vec) {
    if (a.avg) lcnn_pdl::launch(pool_chwn_generic_kernel<4, true>, blocks, kThreads, 0, st, g);
    else lcnn_pdl::launch(pool_chwn_generic_kernel<4, false>, blocks, kThreads, 0, st, g);
  } else {
    if (a.avg) lcnn_pdl::launch(pool_chwn_generic_kernel<1, true>, blocks, kThreads, 0, st, g);
    else lcnn_pdl::launch(pool_chwn_generic_kernel<1, false>, blocks, kThreads, 0, st, g);
  }
  return cudaGetLastError();
}

namespace {

template <int WH, int WW, int S, int FH, int FW>
cudaError_t nchw_launch(const NchwGeom& g, uint32_t blocks, uint32_t smem, bool avg,
                        cudaStream_t st) {
  auto kern = avg ? pool_nchw_kernel<WH, WW, S, FH, FW, true>
                  : pool_nchw_kernel<WH, WW, S, FH, FW, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  lcnn_pdl::launch(kern, blocks, kThreads, smem, st, g);
  return cudaGetLastError();
}

template <int WH, int WW, int S>
bool nchw_dispatch_f(uint32_t fh, uint32_t fw, const NchwGeom& g, uint32_t blocks,
                     uint32_t smem, bool avg, cudaStream_t st, cudaError_t* err) {
#define LCNN_F(FH_, FW_)                                                  \
  if (fh == FH_ && fw == FW_) {                                           \
    *err = nchw_launch<WH, WW, S, FH_, FW_>(g, blocks, smem, avg, st);    \
    return true;                                                          \
  }
  LCNN_F(1, 1) LCNN_F(2, 1) LCNN_F(3, 1) LCNN_F(4, 1)
  LCNN_F(1, 2) LCNN_F(2, 2) LCNN_F(3, 2) LCNN_F(4, 2)
#undef LCNN_F
  return false;
}

}  // namespace

template <int WH, int S, int FH, int FW>
cudaError_t pipe_launch(const NchwPipeGeom& g, uint32_t blocks, uint32_t smem, bool avg,
                        cudaStream_t st) {
  auto kern = avg ? pool_nchw_pipe_kernel<WH, S, FH, FW, true>
                  : pool_nchw_pipe_kernel<WH, S, FH, FW, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  lcnn_pdl::launch_ex(false, kern, blocks, kThreads, smem, st, g);
  return cudaGetLastError();
}

cudaError_t launch_pool_nchw_pipe(const PoolArgs& a, cudaStream_t st) {
  const uint64_t planes = static_cast<uint64_t>(a.n) * a.c;
  const uint64_t row_bytes = static_cast<uint64_t>(a.w) * 4;
  const uint64_t plane_bytes = row_bytes * a.h;
  // Ring slot bytes, slots per CTA and CTAs per SM.  Measured on B200
  // (scripts/nchw_pipe_sweep.sh, profiles/r01_nchw_pipe_sweep.txt): double
  // buffering with more resident CTAs beats a deeper ring -- whole planes
  // (PL5 55x55): 48 KB x 2 x 2 CTAs, 5.26 -> 5.92 TB/s; row bands (VGG):
  // 24 KB x 2 x 4 CTAs, 6.03 -> 6.43 TB/s.  LCNN_NCHW_PIPE="slot_kb,slots,ctas"
  // overrides both (profiling).
  static const uint32_t* knob = [] {
    static uint32_t v[3] = {0, 0, 0};
    if (const char* e = std::getenv("LCNN_NCHW_PIPE"))
      std::sscanf(e, "%u,%u,%u", &v[0], &v[1], &v[2]);
    if (v[1] < 2 || v[1] > kPipeMax) v[0] = 0;
    return v;
  }();
  const bool whole = plane_bytes + 16 <= 48 * 1024;
  uint32_t cfg[3] = {knob[0] ? knob[0] : (whole ? 48u : 24u), knob[0] ? knob[1] : 2u,
                     knob[0] ? knob[2] : (whole ? 2u : 4u)};
  if (a.ring_kb) {  // a tuned ring (lcnn_pool_tune)
    if (a.ring_slots < 2 || a.ring_slots > kPipeMax || !a.ring_ctas) return cudaErrorNotSupported;
    cfg[0] = a.ring_kb;
    cfg[1] = a.ring_slots;
    cfg[2] = a.ring_ctas;
  }
  const uint64_t kSlot = uint64_t{cfg[0]} * 1024;
  if (static_cast<uint64_t>(a.win_h) * row_bytes + 16 > kSlot) return cudaErrorNotSupported;
  if (planes > 0xffffffffull) return cudaErrorNotSupported;
  NchwPipeGeom g;
  g.src = a.src;
  g.dst = a.dst;
  g.H = a.h;
  g.W = a.w;
  g.Ho = a.ho;
  g.Wo = a.wo;
  g.planes = static_cast<uint32_t>(planes);
  g.div_wo = FastDiv((a.wo + a.fw - 1) / a.fw);  // FW-wide output column blocks per row
  g.divisor = static_cast<float>(a.win_h * a.win_w);  // pool.cpp:158
  uint64_t units, span_bytes;
  if (plane_bytes + 16 <= kSlot) {  // whole planes, as many as fit
    g.per_cta = static_cast<uint32_t>((kSlot - 16) / plane_bytes);
    g.band = a.ho;
    g.nbands = 1;
    units = (planes + g.per_cta - 1) / g.per_cta;
    span_bytes = plane_bytes * g.per_cta;
  } else {  // bands of output rows of one plane
    g.per_cta = 1;
    g.band = static_cast<uint32_t>(((kSlot - 16) / row_bytes - a.win_h) / a.stride + 1);
    if (g.band > a.ho) g.band = a.ho;
    g.nbands = (a.ho + g.band - 1) / g.band;
    units = planes * g.nbands;
    span_bytes = (static_cast<uint64_t>(g.band - 1) * a.stride + a.win_h) * row_bytes;
  }
  if (units > 0xffffffffull) return cudaErrorNotSupported;
  g.units = static_cast<uint32_t>(units);
  g.stage_floats = static_cast<uint32_t>((span_bytes + 16 + 15) / 16 * 4);
  const uint32_t nrb = (g.band + a.fh - 1) / a.fh;
  g.div_plane_items = FastDiv(nrb * ((a.wo + a.fw - 1) / a.fw));
  g.pipe = cfg[1];
  const uint32_t smem = g.pipe * g.stage_floats * 4;
  // persistent: cfg[2] CTAs per SM, never more CTAs than units
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t cap = static_cast<uint64_t>(sms) * cfg[2];
  const uint32_t blocks = static_cast<uint32_t>(units < cap ? units : cap);
#define LCNN_PIPE(WH_, S_, FH_, FW_)                                        \
  if (a.win_h == WH_ && a.stride == S_ && a.fh == FH_ && a.fw == FW_)       \
    return pipe_launch<WH_, S_, FH_, FW_>(g, blocks, smem, a.avg, st);
  LCNN_PIPE(2, 2, 1, 1) LCNN_PIPE(2, 2, 2, 1) LCNN_PIPE(2, 2, 3, 1) LCNN_PIPE(2, 2, 4, 1)
  LCNN_PIPE(3, 2, 1, 1) LCNN_PIPE(3, 2, 2, 1) LCNN_PIPE(3, 2, 3, 1) LCNN_PIPE(3, 2, 4, 1)
  LCNN_PIPE(3, 1, 1, 1) LCNN_PIPE(3, 1, 2, 1) LCNN_PIPE(3, 1, 3, 1) LCNN_PIPE(3, 1, 4, 1)
  LCNN_PIPE(2, 2, 1, 2) LCNN_PIPE(2, 2, 2, 2) LCNN_PIPE(2, 2, 4, 2)
  LCNN_PIPE(3, 2, 1, 2) LCNN_PIPE(3, 2, 2, 2) LCNN_PIPE(3, 2, 3, 2) LCNN_PIPE(3, 2, 4, 2)
  LCNN_PIPE(3, 1, 2, 2) LCNN_PIPE(3, 1, 3, 2)
#undef LCNN_PIPE
  return cudaErrorNotSupported;
}

cudaError_t launch_pool_nchw(const PoolArgs& a, cudaStream_t st) {
  const uint64_t planes = static_cast<uint64_t>(a.n) * a.c;
  if (planes == 0 || a.ho == 0 || a.wo == 0) return cudaSuccess;
  if (a.fw <= 2 && a.fh <= 4 && a.win_h == a.win_w &&
      ((a.stride == 2 && (a.win_h == 2 || a.win_h == 3)) || (a.stride == 1 && a.win_h == 3))) {
    const cudaError_t e = launch_pool_nchw_pipe(a, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const uint64_t row_bytes = static_cast<uint64_t>(a.w) * 4;
  // output rows per CTA so that the staged input band fits the budget
  uint32_t band = 1;
  if (static_cast<uint64_t>(a.win_h) * row_bytes <= kStageBudget) {
    const uint64_t rows_fit = kStageBudget / row_bytes;  // >= win_h
    band = static_cast<uint32_t>((rows_fit - a.win_h) / a.stride + 1);
  }
  if (band > a.ho) band = a.ho;
  const uint64_t in_rows = static_cast<uint64_t>(band - 1) * a.stride + a.win_h;
  const uint64_t smem = in_rows * row_bytes + 16;  // + alignment slack
  if (smem > 200 * 1024) {
    const uint64_t total = planes * a.ho * a.wo;
    uint64_t blocks = (total + kThreads - 1) / kThreads;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    const float div = static_cast<float>(a.win_h * a.win_w);
    if (a.avg)
      lcnn_pdl::launch(pool_nchw_direct_kernel<true>, static_cast<uint32_t>(blocks), kThreads, 0, st,
          a.src, a.dst, total, a.h, a.w, a.ho, a.wo, a.win_h, a.win_w, a.stride, div);
    else
      lcnn_pdl::launch(pool_nchw_direct_kernel<false>, static_cast<uint32_t>(blocks), kThreads, 0, st,
          a.src, a.dst, total, a.h, a.w, a.ho, a.wo, a.win_h, a.win_w, a.stride, div);
    return cudaGetLastError();
  }
  NchwGeom g;
  g.src = a.src;
  g.dst = a.dst;
  g.H = a.h;
  g.W = a.w;
  g.Ho = a.ho;
  g.Wo = a.wo;
  g.band = band;
  g.nbands = cdiv(a.ho, band);
  g.divisor = static_cast<float>(a.win_h * a.win_w);  // pool.cpp:158
  g.wh = a.win_h;
  g.ww = a.win_w;
  g.s = a.stride;
  const uint64_t blocks64 = planes * g.nbands;
  if (blocks64 > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const uint32_t blocks = static_cast<uint32_t>(blocks64);
  const uint32_t smem32 = static_cast<uint32_t>(smem);

  cudaError_t err = cudaSuccess;
  g.nbw = cdiv(a.wo, a.fw);
  g.div_nbw = FastDiv(g.nbw);
  bool done = false;
  if (a.win_h == 2 && a.win_w == 2 && a.stride == 2)
    done = nchw_dispatch_f<2, 2, 2>(a.fh, a.fw, g, blocks, smem32, a.avg, st, &err);
  else if (a.win_h == 3 && a.win_w == 3 && a.stride == 2)
    done = nchw_dispatch_f<3, 3, 2>(a.fh, a.fw, g, blocks, smem32, a.avg, st, &err);
  else if (a.win_h == 3 && a.win_w == 3 && a.stride == 1)
    done = nchw_dispatch_f<3, 3, 1>(a.fh, a.fw, g, blocks, smem32, a.avg, st, &err);
  if (done) return err;

  g.nbw = a.wo;
  g.div_nbw = FastDiv(g.nbw);
  auto kern = a.avg ? pool_nchw_generic_kernel<true> : pool_nchw_generic_kernel<false>;
  if (smem32 > 48 * 1024) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem32);
    if (err != cudaSuccess) return err;
  }
  lcnn_pdl::launch(kern, blocks, kThreads, smem32, st, g);
  return cudaGetLastError();
}

cudaError_t launch_pool_oracle(const PoolArgs& a, uint64_t sn, uint64_t sc, uint64_t sh,
                               uint64_t sw, cudaStream_t st) {
  const uint64_t total = static_cast<uint64_t>(a.n) * a.c * a.ho * a.wo;
  if (total == 0) return cudaSuccess;
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  pool_oracle_kernel<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(
      a.src, a.dst, a.n, a.c, a.ho, a.wo, sn, sc, sh, sw, a.win_h, a.win_w, a.stride, a.avg);
  return cudaGetLastError();
}

}  // namespace lcnn_impl
