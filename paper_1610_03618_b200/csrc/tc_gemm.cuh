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

#include <cstdlib>

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
// Loader concept (the producer thread calls begin() once per tile fragment,
// then load() for consecutive (segment, k-block) pairs, so loaders decode K
// incrementally instead of dividing per stage):
//   void prefetch() const;                   // tensor-map prefetch
//   State begin(uint32_t m0, uint32_t n0, uint32_t kfirst) const;
//   void load(State& st, uint32_t seg, uint32_t kb, void* sa, void* sb,
//             uint64_t* bar) const;         // issues TMA, Sched::stage_bytes
//   uint64_t desc_a(const uint8_t* sa, int step) const;  // MMA smem descriptors
//   uint64_t desc_b(const uint8_t* sb, int step) const;  //   of K-step `step`
//   uint32_t resident_bytes() const;        // > 0: B is resident in smem, loaded
//   void load_resident(void* dst, uint64_t* bar) const;  //   once per CTA, and
//   uint32_t resident_offset(uint32_t kb) const;  //  k-block kb's B slice
//   static constexpr bool kZeroSmem;  // stages carry never-loaded zero rows
//   static constexpr bool kResidentA;  // the resident operand is A (else B)
//   static constexpr int kSteps;      // K-steps per stage, 0 = Sched::ksteps
// Segments chain operand sets into one accumulator (3 for 3xTF32).
// Out concept:
//   void store32(uint32_t m, uint32_t n0, const float* v, bool add) const;
//       // row m, columns n0..n0+31; add = stream-K fragment (atomic add)
constexpr int kPBN = 256, kPStages = 4;
constexpr int kPStagesMax = 8;  // ring slots a Sched may ask for (small stages)
constexpr uint32_t kPBBytes = kTcBK * kPBN * 4;            // 32 KB
constexpr uint32_t kPStageBytes = kTcABytes + kPBBytes;    // 48 KB

struct PCtl {
  uint64_t full[kPStagesMax];
  uint64_t empty[kPStagesMax];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t bres;  // resident B operand landed (Loader::resident_bytes() > 0)
  uint32_t tmem_addr;
};
// dynamic shared memory a CTA may opt into on sm_100
constexpr uint32_t kMaxDynSmem = 232448;

// Tile schedule: data-parallel waves of whole tiles, then "stream-K" for the
// ragged last wave.  With T tiles on G resident CTAs, the first
// floor(T/G)*G tiles go round-robin, whole; the k-iterations of the R
// remaining tiles are cut into G equal contiguous ranges, one per CTA, so the
// tail costs R/G of a tile instead of a whole extra wave (and skinny GEMMs
// with T < G -- the fc layers -- are pure stream-K, i.e. an even split-K).
// Fragments of a split tile are combined with 128-bit vector atomic adds
// (red.global.add.v4.f32, resolved in L2, spread over all SMs) into an output
// region the host zeroed beforehand; whole tiles store plainly.  (An owner-
// reduces-partials fixup was measured slower on B200: the single owner CTA
// reading up to ~7 partial tiles serialises the tail, while the reds of all
// fragments proceed in parallel.)  Split-tile sums are therefore not bitwise
// reproducible run to run; the stated tolerances cover any order.
struct Sched {
  uint32_t mt, nt;       // tiles along M, tiles along N (tile t: m = t % mt, n = t / mt)
  uint32_t iters;        // k-iterations per tile (k-blocks x segments)
  uint32_t kbn;          // k-blocks per segment
  uint32_t dp_tiles;     // tiles [0, dp_tiles) are done whole
  uint32_t sk_ctas;      // CTAs sharing the stream-K remainder
  uint64_t sk_iters;     // (tiles - dp_tiles) * iters
  uint32_t grid;         // CTAs to launch
  uint32_t bn;           // N columns of a tile (multiple of 32, <= kPBN)
  uint32_t idesc;        // tcgen05 instruction descriptor (M = 128, N = bn)
  uint32_t stage_bytes;  // TMA bytes per pipeline stage
  uint32_t a_bytes;      // offset of the B operand inside a stage
  uint32_t ksteps;       // MMA K-steps (8 tf32 each) per stage
  uint32_t probe;        // profiling knob (LCNN_TC_PROBE): 1 = no MMAs, 2 = no stores
  // shared-memory carve-up: a ring of `stages` slots of `stage_stride` bytes,
  // then (optionally) the resident B operand at `resident_off`, then PCtl at
  // `ctl_off`; `smem_bytes` is the dynamic allocation (+1 KB for alignment)
  uint32_t stages, stage_stride, resident_off, ctl_off, smem_bytes;
  // epilogue staging for TMA-store outputs (Out::kTmaStore): per epilogue
  // warp epi_bufs 4 KB boxes of 32 rows x 128 B (SWIZZLE_128B) at epi_off
  uint32_t epi_off, epi_bufs;
  // In-kernel zeroing of the stream-K output region (zsync != nullptr; the
  // persistent kernel only): instead of a zero2d launch ahead of the kernel,
  // the epilogue warps of every CTA zero a 1/grid share of the zrows x zwidth
  // words at zp (row pitch zpitch words) right after the PDL wait, then
  // arrive on the caller's two sync words (zsync[0..1], zero before the
  // launch and left zero after it); an epilogue stores into a tile
  // t >= ztile (the first n-tile the region covers) only after all grid
  // arrivals.  Launches sharing the words must never overlap in time.
  unsigned long long* zsync;
  float* zp;
  uint32_t zpitch, zwidth, zrows, ztile;
};

// Out types that write their 32 x 32 accumulator chunks with TMA stores
template <class O, class = void>
struct OutTma {
  static constexpr bool value = false;
};
template <class O>
struct OutTma<O, decltype(void(O::kTmaStore))> {
  static constexpr bool value = O::kTmaStore;
};
// Loaders that prefetch the NEXT layer's constant operand into L2 once this
// CTA's loads are issued (Loader::kTailPrefetch, Loader::tail_prefetch()): the
// fc chain, whose next weights never depend on this layer's output
template <class L, class = void>
struct LoaderTail {
  static constexpr bool value = false;
};
template <class L>
struct LoaderTail<L, decltype(void(L::kTailPrefetch))> {
  static constexpr bool value = L::kTailPrefetch;
};
// Out types whose chunks are staged in pairs (one async-proxy fence per two
// boxes): the short-K SHARE convolutions, where the epilogue sets the pace
// (measured: VGG conv1_1 625 -> 504 us; neutral to slightly slower on the
// long-K layers, whose stores then wait for both previous boxes)
template <class O, class = void>
struct OutTmaPairs {
  static constexpr bool value = false;
};
template <class O>
struct OutTmaPairs<O, decltype(void(O::kTmaPairs))> {
  static constexpr bool value = O::kTmaPairs;
};
// Out types whose tma_quad() stores four consecutive 32-column chunks (128
// columns) of 32 rows as ONE box {32, 4 chunks, 32 rows}: each row's 512 B
// reach memory as one run instead of four 128-B lines written at different
// times (CHWN outputs: a row is a channel plane; profiles/r02_store_pattern_bench.txt)
template <class O, class = void>
struct OutTmaQuads {
  static constexpr bool value = false;
};
template <class O>
struct OutTmaQuads<O, decltype(void(O::kTmaQuads))> {
  static constexpr bool value = O::kTmaQuads;
};
constexpr uint32_t kEpiStageBytes = 4 * 2 * 4096;  // 4 warps x 2 boxes
// Out types that carry state from tile to tile in the epilogue warps'
// registers (Out::Acc) and consume each tile with Out::tile(): the max-pool
// fused into the SHARE convolution, whose CTA walks the conv rows of one
// pooling strip in order (conv.cu SharePoolOut)
template <class O, class = void>
struct OutStateful {
  static constexpr bool value = false;
};
template <class O>
struct OutStateful<O, decltype(void(O::kStateful))> {
  static constexpr bool value = O::kStateful;
};

// One tile's accumulator rows [q*32, q*32+32) (this warp's TMEM lane quarter)
// out of TMEM, 32 columns at a time.  TMA outputs: registers -> a swizzled
// 32 x 128 B shared-memory box -> one TMA store (or f32 add-reduction for a
// stream-K fragment); the box holds the chunk as [row][32 columns]
// (Out::kTmaTransposed = false: rows = accumulator rows) or transposed
// (true: rows = accumulator columns, for outputs whose accumulator rows are
// the contiguous dimension).  Other outputs: Out::store32.
template <class Out>
__device__ __forceinline__ void epilogue_tile(const Out& out, const Sched& sc, uint8_t* stg,
                                              uint32_t taddr, uint32_t m, uint32_t ncol0,
                                              bool split, uint32_t& epi_buf, int lane) {
  if constexpr (OutTmaQuads<Out>::value) {
    if (sc.epi_bufs == 4 && sc.bn % 128 == 0 && !split) {
      // staging [row][chunk][32 floats] (16 KB per warp), SWIZZLE_128B on the
      // box row index row * 4 + chunk; single-buffered
#pragma unroll 1
      for (uint32_t c = 0; c < sc.bn; c += 128) {
        if (lane == 0) bulk_wait_read_n<0>();  // the previous quad's store has read the staging
        __syncwarp();
#pragma unroll 1
        for (uint32_t h = 0; h < 4; ++h) {
          float v[32];
          tmem_ld32(taddr + c + 32 * h, v);
          const uint32_t r = static_cast<uint32_t>(lane) * 4 + h;
          float4* row = reinterpret_cast<float4*>(stg + r * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            row[j ^ (r & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(sc.probe & 2)) {
          out.tma_quad(stg, m, ncol0 + c);
          bulk_commit();
        }
      }
      return;
    }
  }
  if constexpr (OutTmaPairs<Out>::value) {
    if (sc.epi_bufs == 2 && sc.bn % 64 == 0) {
      // pairs of chunks: both boxes written, ONE async-proxy fence, two stores
#pragma unroll 1
      for (uint32_t c = 0; c < sc.bn; c += 64) {
        float v[64];
        tmem_ld32(taddr + c, v);
        tmem_ld32(taddr + c + 32, v + 32);
        if (lane == 0) bulk_wait_read_n<0>();  // both boxes' previous stores have read them
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4* row = reinterpret_cast<float4*>(stg + h * 4096 + lane * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            row[j ^ (lane & 7)] = make_float4(v[32 * h + 4 * j], v[32 * h + 4 * j + 1],
                                              v[32 * h + 4 * j + 2], v[32 * h + 4 * j + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(sc.probe & 2)) {
          out.tma_chunk(stg, m, ncol0 + c, split);
          out.tma_chunk(stg + 4096, m, ncol0 + c + 32, split);
          bulk_commit();
        }
      }
      return;
    }
  }
  if constexpr (OutTma<Out>::value) {
#pragma unroll 1
    for (uint32_t c = 0; c < sc.bn; c += 32) {
      float v[32];
      tmem_ld32(taddr + c, v);
      uint8_t* box = stg + (sc.epi_bufs == 2 ? (epi_buf & 1) : 0u) * 4096;
      ++epi_buf;
      if (lane == 0) {  // this box's previous store has finished reading it
        if (sc.epi_bufs == 2) bulk_wait_read_n<1>();
        else bulk_wait_read_n<0>();
      }
      __syncwarp();
      if constexpr (Out::kTmaTransposed) {
        // column j of the accumulator chunk -> box row j; lane = box column
        const uint32_t col = ((static_cast<uint32_t>(lane) >> 2) << 4) | ((lane & 3) << 2);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          *reinterpret_cast<float*>(box + j * 128 + (col ^ ((j & 7) << 4))) = v[j];
      } else {
        float4* row = reinterpret_cast<float4*>(box + lane * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          row[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && !(sc.probe & 2)) {
        out.tma_chunk(box, m, ncol0 + c, split);
        bulk_commit();
      }
    }
  } else {
#pragma unroll 1
    for (uint32_t c = 0; c < sc.bn; c += 32) {
      float v[32];
      tmem_ld32(taddr + c, v);
      if (!(sc.probe & 2)) out.store32(m, ncol0 + c, v, split);
    }
  }
}

// Default carve-up: kPStages slots of kPStageBytes, no resident operand.
inline void sched_ring(Sched& s, uint32_t stages, uint32_t stride, uint32_t resident_bytes) {
  s.stages = stages;
  s.stage_stride = stride;
  s.resident_off = stages * stride;
  s.ctl_off = (s.resident_off + resident_bytes + 15) / 16 * 16;
  s.smem_bytes = 1024 + s.ctl_off + static_cast<uint32_t>(sizeof(PCtl));
  s.epi_off = 0;
  s.epi_bufs = 0;
}
// Append the TMA-store epilogue staging (1 KB aligned, `bufs` 4 KB boxes per
// epilogue warp) before PCtl.
inline void sched_epi(Sched& s, uint32_t resident_bytes, uint32_t bufs = 2) {
  s.epi_off = (s.resident_off + resident_bytes + 1023) / 1024 * 1024;
  s.epi_bufs = bufs;
  s.ctl_off = s.epi_off + 4 * bufs * 4096;
  s.smem_bytes = 1024 + s.ctl_off + static_cast<uint32_t>(sizeof(PCtl));
}

inline int tc_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || !sms)
      sms = 148;
  }
  return sms;
}

// Fragments shorter than this many k-iterations are not worth an atomic
// epilogue; fewer CTAs then share the remainder.
constexpr uint32_t kMinSkIters = 8;

inline Sched make_sched(uint32_t mt, uint32_t nt, uint32_t kbn, uint32_t segs, uint32_t bn,
                        bool a_mn, bool b_mn, uint32_t min_sk = kMinSkIters, uint32_t units = 0,
                        uint32_t dp_waves = 8) {
  Sched s{};
  s.mt = mt;
  s.nt = nt;
  s.bn = bn;
  s.idesc = idesc_tf32(kTcBM, bn, a_mn, b_mn);
  s.stage_bytes = kTcABytes + bn * kTcBK * 4;
  s.a_bytes = kTcABytes;
  s.ksteps = kTcBK / 8;
  const uint32_t probe = tc_probe_knob();
  s.probe = probe;
  s.kbn = kbn;
  s.iters = kbn * segs;
  const uint32_t tiles = mt * nt;
  const uint32_t g = units ? units : static_cast<uint32_t>(tc_sm_count());
  const uint32_t rem = tiles % g;
  // a last wave that is >= 60% full (or a whole multiple) stays data-parallel:
  // measured on B200, the atomic tail beats an extra wave only below that
  static const bool sk_off = [] {  // profiling knob LCNN_STREAMK=0: whole tiles only
    const char* e = std::getenv("LCNN_STREAMK");
    return e && e[0] == '0';
  }();
  // ... and with >= 8 whole waves the ragged tail is <= 1/9 of the layer:
  // cheaper than zeroing the split tiles' output and reducing fragments
  // (measured on B200: AlexNet conv1, 10.4 waves, 74 -> 68 us)
  static const uint32_t full_pct = [] {  // profiling knob LCNN_SK_FULL_PCT (default 60)
    const char* e = std::getenv("LCNN_SK_FULL_PCT");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 60u;
  }();
  if (rem == 0 || rem * 100 >= g * full_pct || (dp_waves && tiles >= dp_waves * g) || sk_off) {
    s.dp_tiles = tiles;
  } else {
    s.dp_tiles = tiles - rem;
    s.sk_iters = static_cast<uint64_t>(rem) * s.iters;
    uint64_t c = s.sk_iters / min_sk;
    s.sk_ctas = static_cast<uint32_t>(c < 1 ? 1 : (c > g ? g : c));
  }
  const uint32_t dp_grid = s.dp_tiles < g ? s.dp_tiles : g;
  s.grid = dp_grid > s.sk_ctas ? dp_grid : s.sk_ctas;
  sched_ring(s, kPStages, kPStageBytes, 0);
  return s;
}

// First column of the stream-K region; the host zeroes every column from
// there on (whole tiles in that range are overwritten by plain stores).
inline uint32_t sched_zero_col(const Sched& s, uint32_t bn) {
  return s.dp_tiles == s.mt * s.nt ? ~0u : (s.dp_tiles / s.mt) * bn;
}

// Zero the stream-K output region (rows x width words at p, row pitch
// `pitch` words, covering the tiles from `first_tile` on): in the persistent
// kernel itself when the caller owns a sync word (Sched::zsync), else as a
// zero2d launch ahead of it.  The launcher (zero2d) is passed in so that this
// header stays free of the host library.
template <class ZeroFn>
inline cudaError_t sched_zero_region(Sched& s, unsigned long long* sync, float* p,
                                     uint64_t pitch, uint64_t width, uint64_t rows,
                                     uint32_t first_tile, ZeroFn&& zero2d) {
  if (!width || !rows) return cudaSuccess;
  const bool fits = pitch < (1ull << 32) && width * rows < (1ull << 31);
  if (sync && fits) {
    s.zsync = sync;
    s.zp = p;
    s.zpitch = static_cast<uint32_t>(pitch);
    s.zwidth = static_cast<uint32_t>(width);
    s.zrows = static_cast<uint32_t>(rows);
    s.ztile = first_tile;
    return cudaSuccess;
  }
  return zero2d(p, pitch, width, rows);
}

// Calls f(tile, kbeg, kend, split) for work unit `id` of `count` (a CTA, or
// a CTA pair), in order.
template <class F>
__device__ __forceinline__ void for_each_work(const Sched& s, uint32_t id, uint32_t count, F&& f) {
  for (uint32_t t = id; t < s.dp_tiles; t += count) f(t, 0u, s.iters, false);
  if (id < s.sk_ctas) {
    uint64_t lo = s.sk_iters * id / s.sk_ctas;
    const uint64_t hi = s.sk_iters * (id + 1) / s.sk_ctas;
    while (lo < hi) {
      const uint32_t tr = static_cast<uint32_t>(lo / s.iters);
      const uint64_t base = static_cast<uint64_t>(tr) * s.iters;
      const uint32_t kb = static_cast<uint32_t>(lo - base);
      const uint32_t ke = static_cast<uint32_t>(hi - base < s.iters ? hi - base : s.iters);
      f(s.dp_tiles + tr, kb, ke, !(kb == 0 && ke == s.iters));
      lo = base + ke;
    }
  }
}
template <class F>
__device__ __forceinline__ void for_each_work(const Sched& s, F&& f) {
  for_each_work(s, blockIdx.x, gridDim.x, static_cast<F&&>(f));
}

// In-kernel zeroing (Sched::zsync): sync[0] counts the CTAs that zeroed
// their share, sync[1] the CTAs that finished; the last CTA to finish resets
// both, so the words are zero again for the next launch of the call site
// (whatever its grid size).  Epilogue warps (2..5) of every CTA zero this
// CTA's 1/grid share of the region and arrive.
__device__ __forceinline__ void zero_region_arrive(const Sched& sc) {
  const uint32_t tid = threadIdx.x - 64, G = gridDim.x;
  const bool vec = ((sc.zwidth | sc.zpitch) & 3u) == 0 && (reinterpret_cast<uintptr_t>(sc.zp) & 15u) == 0;
  const uint32_t w = vec ? sc.zwidth / 4 : sc.zwidth;
  const uint32_t total = w * sc.zrows;  // host guarantees < 2^31
  const uint32_t lo = static_cast<uint32_t>(static_cast<uint64_t>(total) * blockIdx.x / G);
  const uint32_t hi = static_cast<uint32_t>(static_cast<uint64_t>(total) * (blockIdx.x + 1) / G);
  for (uint32_t i = lo + tid; i < hi; i += 128) {
    const uint32_t r = i / w, c = i - r * w;
    if (vec)
      reinterpret_cast<float4*>(sc.zp + static_cast<uint64_t>(r) * sc.zpitch)[c] =
          make_float4(0.f, 0.f, 0.f, 0.f);
    else
      sc.zp[static_cast<uint64_t>(r) * sc.zpitch + c] = 0.0f;
  }
  // the stream-K fragments land through the async proxy (TMA add-reductions)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (tid == 0) {
    __threadfence();
    atomicAdd(sc.zsync, 1ull);
  }
}
// An epilogue warp waits until every CTA of the grid zeroed its share
// (acquire), before its first store into the region.
__device__ __forceinline__ void zero_region_wait(const unsigned long long* sync, int lane) {
  if (lane == 0) {
    const unsigned long long G = gridDim.x;
    unsigned long long v;
    for (uint32_t spins = 0;; ++spins) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(sync) : "memory");
      if (v >= G) break;
      // every CTA of the grid is resident (grid <= SMs, one CTA per SM), so
      // the arrivals come within microseconds; seconds mean a CTA can never
      // be scheduled (e.g. SMs withheld from the context): fail loudly
      if (spins > (1u << 26)) __trap();
      __nanosleep(64);
    }
  }
  __syncwarp();
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// One thread per CTA after the CTA's last store: the grid's last CTA resets
// both words (every CTA has passed its wait by then).
__device__ __forceinline__ void zero_region_depart(unsigned long long* sync) {
  if (atomicAdd(sync + 1, 1ull) == gridDim.x - 1ull) {
    atomicExch(sync, 0ull);
    atomicExch(sync + 1, 0ull);
  }
}

template <class Loader, class Out>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_persistent(const __grid_constant__ Loader ld, const __grid_constant__ Out out,
                       const __grid_constant__ Sched sc) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  PCtl* ctl = reinterpret_cast<PCtl*>(smem + sc.ctl_off);
  const uint32_t nst = sc.stages;
  const uint32_t res_bytes = ld.resident_bytes();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if constexpr (Loader::kZeroSmem) {
    // K padding rows that no TMA box ever writes must read as zeros
    float4* z = reinterpret_cast<float4*>(smem);
    for (uint32_t i = threadIdx.x; i < sc.ctl_off / 16; i += blockDim.x)
      z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    if (lane == 0) {
      ld.prefetch();
      for (uint32_t s = 0; s < nst; ++s) {
        mbar_init(&ctl->full[s], 1);
        mbar_init(&ctl->empty[s], 1);
      }
      mbar_init(&ctl->bres, 1);
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
  LCNN_PDL_ENTRY();  // the prologue above overlapped the previous kernel's tail

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    if (res_bytes) {  // the B operand every tile of this CTA uses, loaded once
      mbar_arrive_expect_tx(&ctl->bres, res_bytes);
      ld.load_resident(smem + sc.resident_off, &ctl->bres);
    }
    uint32_t s = 0, phase = 0;
    for_each_work(sc, [&](uint32_t t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t ntile = t / sc.mt;
      uint32_t seg = kbeg / sc.kbn, kb = kbeg - seg * sc.kbn;
      auto st = ld.begin((t - ntile * sc.mt) * kTcBM, ntile * sc.bn, kb);

      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->empty[s], phase ^ 1);
        uint8_t* sa = smem + s * sc.stage_stride;
        mbar_arrive_expect_tx(&ctl->full[s], sc.stage_bytes);
        ld.load(st, seg, kb, sa, sa + sc.a_bytes, &ctl->full[s]);
        if (++kb == sc.kbn) {
          kb = 0;
          ++seg;
        }
        if (++s == nst) {
          s = 0;
          phase ^= 1;
        }
      }
    });
    if constexpr (LoaderTail<Loader>::value) ld.tail_prefetch(blockIdx.x, gridDim.x);
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp walks the schedule (warp-uniform control flow keeps the
    // descriptor arithmetic on the uniform datapath); one elected lane issues
    // the MMAs and commits.  Every Loader's descriptors are affine in the
    // K-step, so a stage needs two base descriptors and the per-step
    // increments are kernel constants (the issue loop is then ~1 add per
    // operand per MMA: at ~26 dependent instructions per MMA the issuing
    // thread, not the tensor core, set the pace of narrow-K stages).
    const uint32_t idesc = sc.idesc;
    const uint64_t dai = ld.desc_a(smem, 1) - ld.desc_a(smem, 0);
    const uint64_t dbi = ld.desc_b(smem, 1) - ld.desc_b(smem, 0);
    const uint32_t ksteps = Loader::kSteps > 0 ? static_cast<uint32_t>(Loader::kSteps) : sc.ksteps;
    const bool mma_on = !(sc.probe & 1);
    uint32_t s = 0, phase = 0, local = 0;
    if (res_bytes) {
      mbar_wait(&ctl->bres, 0);
      tc_fence_after();
    }
    for_each_work(sc, [&](uint32_t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      mbar_wait(&ctl->tempty[a], aphase ^ 1);  // epilogue drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + a * kPBN;
      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->full[s], phase);
        tc_fence_after();
        const uint8_t* slot = smem + s * sc.stage_stride;
        // resident operand (B, or A when Loader::kResidentA): the slice of
        // k-block `it` (single segment when resident)
        const uint8_t* sres =
            res_bytes ? smem + sc.resident_off + ld.resident_offset(it % sc.kbn) : nullptr;
        const uint8_t* sa = Loader::kResidentA && res_bytes ? sres : slot;
        const uint8_t* sb = Loader::kResidentA || !res_bytes ? slot + sc.a_bytes : sres;
        const uint64_t da = ld.desc_a(sa, 0), db = ld.desc_b(sb, 0);
        if (elect_one()) {
          if (mma_on) {
            mma_tf32(acc, da, db, idesc, it != kbeg);
            uint64_t xa = da, xb = db;
            if constexpr (Loader::kSteps > 0) {
#pragma unroll
              for (int k = 1; k < Loader::kSteps; ++k) {
                xa += dai;
                xb += dbi;
                mma_tf32(acc, xa, xb, idesc, 1u);
              }
            } else {
#pragma unroll 1
              for (uint32_t k = 1; k < ksteps; ++k) {
                xa += dai;
                xb += dbi;
                mma_tf32(acc, xa, xb, idesc, 1u);
              }
            }
          }
          tc_commit(&ctl->empty[s]);
        }
        __syncwarp();
        if (++s == nst) {
          s = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) tc_commit(&ctl->tfull[a]);
      __syncwarp();
    });
  } else if (warp >= 2) {
    // ---------------- stateful epilogue (Out::tile) ----------------
    if constexpr (OutStateful<Out>::value) {
      const int q = warp & 3;
      uint32_t local = 0, epi_buf = 0;
      typename Out::Acc acc;
      for_each_work(sc, [&](uint32_t t, uint32_t, uint32_t, bool) {
        const uint32_t a = local & 1, aphase = (local >> 1) & 1;
        ++local;
        mbar_wait(&ctl->tfull[a], aphase);
        tc_fence_after();
        const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
        out.tile(acc, t, base, smem + sc.epi_off + q * sc.epi_bufs * 4096, epi_buf, q, lane);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->tempty[a]);
      });
      if (lane == 0) bulk_wait_read_n<0>();
    } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    uint32_t local = 0, epi_buf = 0;
    bool zwait = sc.zsync != nullptr;
    if (zwait) zero_region_arrive(sc);
    for_each_work(sc, [&](uint32_t t, uint32_t, uint32_t, bool split) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      const uint32_t ntile = t / sc.mt;
      mbar_wait(&ctl->tfull[a], aphase);
      tc_fence_after();
      if (zwait && t >= sc.ztile) {
        zero_region_wait(sc.zsync, lane);
        zwait = false;
      }
      const uint32_t m = (t - ntile * sc.mt) * kTcBM + q * 32 + lane;
      const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
      epilogue_tile(out, sc, smem + sc.epi_off + q * sc.epi_bufs * 4096, base, m, ntile * sc.bn,
                    split, epi_buf, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl->tempty[a]);
    });
    if constexpr (OutTma<Out>::value) {
      if (lane == 0) bulk_wait_read_n<0>();
    }
    }
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

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs (one TPC)
// computes 256-row tiles (UMMA M = 256).  Each CTA loads its own 128 A rows
// and HALF of the tile's B columns, so an SM ingests A + B/2 per stage
// instead of A + B -- the lever for layers whose TMA delivery, not the tensor
// pipe, sets the pace (conv2-5: filters are ~60% of each stage).  The leader
// (rank 0) waits for both CTAs' bytes on its own full barrier (TMA
// .cta_group::2 completes on a peer-CTA mbarrier), issues the M = 256 MMAs
// and multicasts its commits to both CTAs' empty / tfull barriers; each CTA's
// epilogue drains its own TMEM half and arrives on the leader's tempty.
// Loader contract as above, plus: begin() receives this CTA's A-row and
// B-column origins, and load() completes on the LEADER's barrier.
template <class Loader, class Out>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    tc_gemm_pair(const __grid_constant__ Loader ld, const __grid_constant__ Out out,
                 const __grid_constant__ Sched sc) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  PCtl* ctl = reinterpret_cast<PCtl*>(smem + sc.ctl_off);
  const uint32_t nst = sc.stages;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0) {
    if (lane == 0) {
      ld.prefetch();
      for (uint32_t s = 0; s < nst; ++s) {
        mbar_init(&ctl->full[s], 1);
        mbar_init(&ctl->empty[s], 1);
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
  cluster_sync();  // the peer's barriers exist before any remote arrive or TMA completion
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_addr;
  LCNN_PDL_ENTRY();
  const uint32_t half_bn = sc.bn / 2;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    uint32_t s = 0, phase = 0;
    for_each_work(sc, pair, npairs, [&](uint32_t t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t ntile = t / sc.mt;
      uint32_t seg = kbeg / sc.kbn, kb = kbeg - seg * sc.kbn;
      auto st = ld.begin((t - ntile * sc.mt) * (2 * kTcBM) + rank * kTcBM,
                         ntile * sc.bn + rank * half_bn, kb);
      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->empty[s], phase ^ 1);
        uint8_t* sa = smem + s * sc.stage_stride;
        if (rank == 0) mbar_arrive_expect_tx(&ctl->full[s], 2 * sc.stage_bytes);
        ld.load(st, seg, kb, sa, sa + sc.a_bytes, &ctl->full[s]);
        if (++kb == sc.kbn) {
          kb = 0;
          ++seg;
        }
        if (++s == nst) {
          s = 0;
          phase ^= 1;
        }
      }
    });
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader) ----------------
    const uint32_t idesc = sc.idesc;
    const uint64_t dai = ld.desc_a(smem, 1) - ld.desc_a(smem, 0);
    const uint64_t dbi = ld.desc_b(smem, 1) - ld.desc_b(smem, 0);
    const bool mma_on = !(sc.probe & 1);
    uint32_t s = 0, phase = 0, local = 0;
    for_each_work(sc, pair, npairs, [&](uint32_t, uint32_t kbeg, uint32_t kend, bool) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      mbar_wait(&ctl->tempty[a], aphase ^ 1);  // both epilogues drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + a * kPBN;
      for (uint32_t it = kbeg; it < kend; ++it) {
        mbar_wait(&ctl->full[s], phase);
        tc_fence_after();
        const uint8_t* sa = smem + s * sc.stage_stride;
        const uint64_t da = ld.desc_a(sa, 0), db = ld.desc_b(sa + sc.a_bytes, 0);
        if (elect_one()) {
          if (mma_on) {
            mma_tf32_cg2(acc, da, db, idesc, it != kbeg);
            uint64_t xa = da, xb = db;
#pragma unroll
            for (int k = 1; k < Loader::kSteps; ++k) {
              xa += dai;
              xb += dbi;
              mma_tf32_cg2(acc, xa, xb, idesc, 1u);
            }
          }
          tc_commit_cg2(&ctl->empty[s], 3);
        }
        __syncwarp();
        if (++s == nst) {
          s = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) tc_commit_cg2(&ctl->tfull[a], 3);
      __syncwarp();
    });
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs: own TMEM half) ----------------
    const int q = warp & 3;
    const uint32_t leader_tempty = mapa_shared(smem_u32(&ctl->tempty[0]), 0);
    uint32_t local = 0, epi_buf = 0;
    for_each_work(sc, pair, npairs, [&](uint32_t t, uint32_t, uint32_t, bool split) {
      const uint32_t a = local & 1, aphase = (local >> 1) & 1;
      ++local;
      const uint32_t ntile = t / sc.mt;
      mbar_wait(&ctl->tfull[a], aphase);
      tc_fence_after();
      const uint32_t m = (t - ntile * sc.mt) * (2 * kTcBM) + rank * kTcBM + q * 32 + lane;
      const uint32_t base = tmem + a * kPBN + (static_cast<uint32_t>(q * 32) << 16);
      epilogue_tile(out, sc, smem + sc.epi_off + q * sc.epi_bufs * 4096, base, m, ntile * sc.bn,
                    split, epi_buf, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + a * 8);
    });
    if constexpr (OutTma<Out>::value) {
      if (lane == 0) bulk_wait_read_n<0>();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem);
  }
}

// Shared store of 32 consecutive accumulator columns of one row: plain
// 128-bit stores for whole tiles, vector atomic adds for stream-K fragments.
__device__ __forceinline__ void store_row32(float* row, uint32_t n0, uint32_t N, const float* v,
                                            bool add) {
  if (n0 + 32 <= N && (reinterpret_cast<uintptr_t>(row) & 15u) == 0) {
    if (add) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        atomicAdd(reinterpret_cast<float4*>(row + j),
                  make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(row + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < N) {
        if (add)
          atomicAdd(row + j, v[j]);
        else
          row[j] = v[j];
      }
  }
}

// Warp-cooperative store of 32 rows x 32 consecutive floats (lane = row, v =
// its 32 accumulator columns) -- the channels-on-M epilogue, where a row is
// an output channel and consecutive rows are far apart in memory.  Stored
// lane by lane, every instruction would touch 32 lines with 16 B each; here
// an 8 x 8 butterfly of 16-B chunks inside each 8-lane group (3 rounds of
// shfl.xor) first gives lane l of group q chunk l of rows 8q..8q+7, so each
// of the 8 store instructions writes 4 whole 128-byte lines.  rowp: this
// lane's row start (16-B aligned) or nullptr to skip the row.  add: vector
// atomic adds (stream-K fragments) -- those stay row-per-lane (one 16-B red
// per line per instruction spreads over more L2 atomic units than 8 lanes
// adding into the same line; measured on the fc layers).  All 32 lanes must
// call it.
__device__ __forceinline__ void warp_store_rows32(float* rowp, const float* v, bool add) {
  if (add) {
    if (rowp) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        atomicAdd(reinterpret_cast<float4*>(rowp + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
    }
    return;
  }
  const uint32_t lane = threadIdx.x & 31, l8 = lane & 7, q8 = lane & ~7u;
  float4 x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
#pragma unroll
  for (int b = 1; b < 8; b <<= 1) {
    const bool hi = (l8 & b) != 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j & b) continue;
      const float4 send = hi ? x[j] : x[j | b];
      float4 r;
      r.x = __shfl_xor_sync(0xffffffffu, send.x, b);
      r.y = __shfl_xor_sync(0xffffffffu, send.y, b);
      r.z = __shfl_xor_sync(0xffffffffu, send.z, b);
      r.w = __shfl_xor_sync(0xffffffffu, send.w, b);
      if (hi)
        x[j] = r;
      else
        x[j | b] = r;
    }
  }
  const unsigned long long mine = reinterpret_cast<unsigned long long>(rowp);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float* p = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, mine, q8 + j));
    if (!p) continue;
    lcnn_tc::st_out(reinterpret_cast<float4*>(p) + l8, x[j]);
  }
}

// ---------------------------------------------------------------------------
// Cluster split-K for skinny GEMMs (the fc layers: M = one batch of 128
// rows): one output tile per cluster of S CTAs, CTA r accumulating the r-th
// of S equal k-ranges in its own TMEM.  The S partial tiles are then summed
// through distributed shared memory -- each CTA parks its fragment in its
// (now idle) pipeline ring, and after a cluster barrier CTA r reduces rows
// [r*128/S, (r+1)*128/S) of the tile by reading all S fragments over DSMEM
// and writes them once with coalesced 128-bit stores.  No atomics, no
// pre-zeroed output (so no memset node in the layer chain), and the sums are
// bitwise reproducible (fixed order r = 0..S-1).
struct SplitK {
  uint32_t mt, nt;     // tiles along M (128 rows) and N (bn columns)
  uint32_t iters;      // k-iterations per tile (k-blocks x segments)
  uint32_t kbn;        // k-blocks per segment
  uint32_t S;          // CTAs per cluster = k-ranges per tile
  uint32_t bn, idesc, stage_bytes, a_bytes;
  uint32_t stages, stage_stride, ctl_off, smem_bytes;
  uint32_t M, N;       // output extents (row-major C, ldc = N)
  uint32_t probe;
};
constexpr uint32_t kSplitPitch = kPBN + 4;  // fragment row pitch in floats (16-B skew per row)

template <class Loader>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_splitk(const __grid_constant__ Loader ld, float* __restrict__ c,
                   const __grid_constant__ SplitK sk) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  PCtl* ctl = reinterpret_cast<PCtl*>(smem + sk.ctl_off);
  const uint32_t nst = sk.stages;
  const uint32_t rank = cluster_ctarank();
  const uint32_t tile = blockIdx.x / sk.S;
  const uint32_t ntile = tile / sk.mt, m0 = (tile - ntile * sk.mt) * kTcBM, n0 = ntile * sk.bn;
  const uint32_t kbeg = static_cast<uint32_t>(static_cast<uint64_t>(sk.iters) * rank / sk.S);
  const uint32_t kend = static_cast<uint32_t>(static_cast<uint64_t>(sk.iters) * (rank + 1) / sk.S);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0) {
    if (lane == 0) {
      ld.prefetch();
      for (uint32_t s = 0; s < nst; ++s) {
        mbar_init(&ctl->full[s], 1);
        mbar_init(&ctl->empty[s], 1);
      }
      mbar_init(&ctl->tfull[0], 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc<256>(&ctl->tmem_addr);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_addr;
  LCNN_PDL_ENTRY();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    uint32_t s = 0, phase = 0;
    uint32_t seg = kbeg / sk.kbn, kb = kbeg - seg * sk.kbn;
    auto st = ld.begin(m0, n0, kb);
    for (uint32_t it = kbeg; it < kend; ++it) {
      mbar_wait(&ctl->empty[s], phase ^ 1);
      uint8_t* sa = smem + s * sk.stage_stride;
      mbar_arrive_expect_tx(&ctl->full[s], sk.stage_bytes);
      ld.load(st, seg, kb, sa, sa + sk.a_bytes, &ctl->full[s]);
      if (++kb == sk.kbn) {
        kb = 0;
        ++seg;
      }
      if (++s == nst) {
        s = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform, one elected lane) ----------------
    const uint64_t dai = ld.desc_a(smem, 1) - ld.desc_a(smem, 0);
    const uint64_t dbi = ld.desc_b(smem, 1) - ld.desc_b(smem, 0);
    uint32_t s = 0, phase = 0;
    for (uint32_t it = kbeg; it < kend; ++it) {
      mbar_wait(&ctl->full[s], phase);
      tc_fence_after();
      const uint8_t* sa = smem + s * sk.stage_stride;
      const uint64_t da = ld.desc_a(sa, 0), db = ld.desc_b(sa + sk.a_bytes, 0);
      if (elect_one()) {
        if (!(sk.probe & 1)) {
          mma_tf32(tmem, da, db, sk.idesc, it != kbeg);
          uint64_t xa = da, xb = db;
#pragma unroll
          for (int k = 1; k < Loader::kSteps; ++k) {
            xa += dai;
            xb += dbi;
            mma_tf32(tmem, xa, xb, sk.idesc, 1u);
          }
        }
        tc_commit(&ctl->empty[s]);
      }
      __syncwarp();
      if (++s == nst) {
        s = 0;
        phase ^= 1;
      }
    }
    if (elect_one()) tc_commit(&ctl->tfull[0]);
    __syncwarp();
  } else if (warp >= 2) {
    // ---------------- park the fragment in the idle ring ----------------
    // (every MMA -- the ring's last reader -- completed before tfull fires)
    const int q = warp & 3;
    mbar_wait(&ctl->tfull[0], 0);
    tc_fence_after();
    float* frag = reinterpret_cast<float*>(smem);
    const uint32_t row = q * 32 + lane;
    const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
    for (uint32_t col = 0; col < sk.bn; col += 32) {
      float v[32];
      tmem_ld32(base + col, v);
      if (kend == kbeg || (sk.probe & 1)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
      }
      float4* d = reinterpret_cast<float4*>(frag + row * kSplitPitch + col);
#pragma unroll
      for (int j = 0; j < 8; ++j) d[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every fragment of the cluster is parked
  // ---------------- DSMEM reduction: rows [rank*128/S, (rank+1)*128/S) ----------------
  {
    const uint32_t r0 = kTcBM * rank / sk.S, r1 = kTcBM * (rank + 1) / sk.S;
    const uint32_t q4 = sk.bn / 4;  // float4 per row
    const uint32_t frag0 = smem_u32(smem);
    uint32_t src[16];
    for (uint32_t j = 0; j < sk.S; ++j) src[j] = mapa_shared(frag0, j);
    const bool vec = (sk.N % 4) == 0;
    for (uint32_t i = threadIdx.x; i < (r1 - r0) * q4; i += blockDim.x) {
      const uint32_t rr = r0 + i / q4, c4 = i % q4;
      const uint32_t off = (rr * kSplitPitch + c4 * 4) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t j = 0; j < sk.S; ++j) {
        float4 v;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(src[j] + off));
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      const uint32_t m = m0 + rr, n = n0 + c4 * 4;
      if (m >= sk.M || n >= sk.N || (sk.probe & 2)) continue;
      float* dst = c + static_cast<uint64_t>(m) * sk.N + n;
      if (vec && n + 4 <= sk.N) {
        lcnn_tc::st_out(reinterpret_cast<float4*>(dst), acc);
      } else {
        const float a[4] = {acc.x, acc.y, acc.z, acc.w};
        for (uint32_t e = 0; e < 4 && n + e < sk.N; ++e) dst[e] = a[e];
      }
    }
  }
  cluster_sync();  // peers finished reading this CTA's fragment
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

template <class Loader>
cudaError_t launch_splitk(const Loader& ld, float* c, const SplitK& sk, cudaStream_t s) {
  auto kern = tc_gemm_splitk<Loader>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (sk.smem_bytes > kMaxDynSmem || sk.stages < 2 || sk.stages > kPStagesMax || sk.S < 1 ||
      sk.S > 16)
    return cudaErrorInvalidConfiguration;
  static bool nonportable = false;
  if (sk.S > 8 && !nonportable) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    nonportable = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sk.mt * sk.nt * sk.S);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = sk.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = sk.S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = lcnn_pdl::enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, ld, c, sk);
}

template <class Loader, class Out>
cudaError_t launch_pair(const Loader& ld, const Out& out, const Sched& sc, cudaStream_t s) {
  auto kern = tc_gemm_pair<Loader, Out>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // the pair kernel has no in-kernel zeroing (Sched::zsync)
  if (sc.smem_bytes > kMaxDynSmem || sc.stages < 2 || sc.stages > kPStagesMax || sc.grid % 2 ||
      sc.zsync)
    return cudaErrorInvalidConfiguration;
  return lcnn_pdl::launch(kern, sc.grid, kTcThreads, sc.smem_bytes, s, ld, out, sc);
}

// Host launch of the persistent kernel (one dynamic-smem opt-in per
// Loader/Out instantiation).
template <class Loader, class Out>
cudaError_t launch_persistent(const Loader& ld, const Out& out, const Sched& sc, cudaStream_t s) {
  auto kern = tc_gemm_persistent<Loader, Out>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (sc.smem_bytes > kMaxDynSmem || sc.stages < 2 || sc.stages > kPStagesMax ||
      (OutStateful<Out>::value && sc.zsync))  // stateful epilogues never split tiles
    return cudaErrorInvalidConfiguration;
  return lcnn_pdl::launch(kern, sc.grid, kTcThreads, sc.smem_bytes, s, ld, out, sc);
}

}  // namespace lcnn_tc
