// Softmax classifier on sm_100a: the fused single kernel and the five-kernel
// multi-pass baseline.
//
// Reference: /root/reference/proj/src/softmax.cpp
//   softmax_reference :36-98   max; x-max -> midv1; exp -> midv2; blocked sum;
//                              x (1/sum)  (8 full-matrix sweeps, 3 arrays)
//   softmax_fused     :100-145 row staged once, blocked max then exp+sum,
//                              out = e * (1/sum)  (2 sweeps)
//   streaming         :146-178 rows wider than the local buffer
//   check_finite      :15-19   DomainError on inf/NaN
// Paper: PAPER.md Fig. 9 (one kernel, shared-memory reductions).
//
// Numerics: the fused kernels take e^(x - max) on the SFU (fexp below:
// ex2.approx of (x - max) * log2(e)), inv = 1/sum in IEEE division, out =
// e * inv.  Against the reference's libm expf that is <= ~1e-7 relative per
// exponential and <= 2.2e-8 absolute from rounding the scaled argument,
// inside the parity bound approx_equal 1e-6 (tensor.cpp:157-187; outputs are
// <= 1, so the bound is 1e-6 absolute).  With accurate expf (~20
// instructions) the 4096 x 1000 classifier was instruction-issue-bound at
// ~3.6 us of its ~10 us (now 7.5 us).  A shared-memory-staged variant (bulk
// copies in and out, per-chunk mbarriers) measured slower (9.4 us): the
// register-resident kernel with 32 warps per SM keeps more requests in
// flight.  The reduction order (parallel tree vs the CPU's 256-blocked sum)
// is the other difference.  The five-kernel baseline keeps
// accurate expf, as the reference's softmax_reference does.
//
// Fused kernel shapes (all one launch, one HBM read + one HBM write):
//   cols <= 2048      : LPR lanes per row (4..32), values held in registers,
//                       128-bit loads when cols % 4 == 0, shuffle reductions;
//   cols <= 16384     : one CTA (256 threads) per row, registers + a
//                       shared-memory cross-warp reduction;
//   wider             : one CTA per row, online (max, sum) pass then a
//                       normalise pass (input read twice).
#include <float.h>

#include <cstdlib>

#include <cuda.h>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace lcnn_dev {

// e^d on the SFU: ex2.approx.ftz(d * log2 e)
__device__ __forceinline__ float fexp(float d) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d * 1.4426950408889634f));
  return r;
}

// Blackwell packed fp32 pairs (FADD2 / FMUL2 / FFMA2: two lanes of work per
// issue slot; PTX .f32x2, sm_100+)
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float ex2_sfu(float t) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
  return r;
}

__device__ __forceinline__ void flag_nonfinite(int* flag, bool bad) {
  if (bad && flag) *reinterpret_cast<volatile int*>(flag) = 1;
}

template <int LPR>
__device__ __forceinline__ float group_max(float v, unsigned mask) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(mask, v, o));
  return v;
}
template <int LPR>
__device__ __forceinline__ float group_sum(float v, unsigned mask) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// LPR lanes own one row; each lane holds VPL values.  Capped at 64 registers
// (32 warps per SM) so a 4096-row batch runs in a single wave; 128-thread
// CTAs (4 rows of 1000) spread that wave evenly -- 1024 CTAs place 6-7 per
// SM (27-28 rows) where 512 256-thread CTAs placed 3-4 (24-32 rows).
//
// Per element the kernel issues 7 instructions: max, min (the finiteness
// test), x - m, the log2e scale and MUFU.EX2, the sum add and the final
// scale.  ncu on the 4096 x 1000 classifier (round 2) showed the schedulers
// at 42 % issue with ~530 instructions per row (per-element bounds
// predicates and an isfinite test per element), so the short single wave
// was issue-limited as much as latency-limited.  Slots past the row end hold
// -FLT_MAX: neutral for the max, invisible to the min test, e^-inf = 0 in
// the sum.  Non-finite detection: +inf -> max = inf, -inf -> min = -inf, NaN
// -> the sum is NaN (fmaxf / fminf skip NaN, the exponential does not).
// (VPL = 64, rows of up to 2048: 128 registers, 16 warps per SM -- at the
// 64-register cap those 64 values spilled ~370 bytes per thread)
template <int LPR, int VPL, bool VEC, int THREADS = kThreads>
__global__ void __launch_bounds__(THREADS, (VPL > 32 ? 512 : 1024) / THREADS)
    softmax_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                        uint32_t rows, uint32_t cols, int* flag) {
  LCNN_PDL_ENTRY();
  constexpr int kGroups = THREADS / LPR;
  static_assert(VPL % 2 == 0, "values are processed in fp32 pairs");
  const uint32_t row = blockIdx.x * kGroups + threadIdx.x / LPR;
  const int lane = threadIdx.x % LPR;
  const int wl = threadIdx.x & 31;
  const unsigned mask =
      LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (wl & ~(LPR - 1)));
  if (row >= rows) return;  // uniform per group
  const float* in = src + static_cast<uint64_t>(row) * cols;
  float* out = dst + static_cast<uint64_t>(row) * cols;

  float v[VPL];
  if constexpr (VEC) {
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k) {
      const uint32_t col = (lane + k * LPR) * 4;
      if (col < cols) {
        const float4 q = ldg_stream(reinterpret_cast<const float4*>(in + col));
        v[4 * k + 0] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
      } else {
        v[4 * k + 0] = v[4 * k + 1] = v[4 * k + 2] = v[4 * k + 3] = -FLT_MAX;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t col = lane + k * LPR;
      v[k] = col < cols ? __ldg(in + col) : -FLT_MAX;
    }
  }
  float m = -FLT_MAX, mn = FLT_MAX;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    m = fmaxf(m, v[k]);
    mn = fminf(mn, v[k]);
  }
  const bool neg_inf = !(mn >= -FLT_MAX);
  m = group_max<LPR>(m, mask);
  // pairs: t = (x - m) * log2e with FADD2 + FMUL2, e = 2^t on the SFU, sums
  // kept as a pair.  (2^t on the FMA pipe for every 2nd / 4th pair -- a
  // degree-5 polynomial -- measured slower on B200: 4096 x 1000 6.39 ->
  // 6.45 / 6.47 us; the SFU is not what bounds this kernel.)
  const unsigned long long mm = f2_pack(m, m);
  const unsigned long long l2e = f2_pack(1.4426950408889634f, 1.4426950408889634f);
  unsigned long long s2 = 0ull;  // (+0.0f, +0.0f)
#pragma unroll
  for (int k = 0; k < VPL / 2; ++k) {
    float t0, t1, e0, e1;
    f2_unpack(f2_mul(f2_sub(f2_pack(v[2 * k], v[2 * k + 1]), mm), l2e), t0, t1);
    e0 = ex2_sfu(t0);
    e1 = ex2_sfu(t1);
    v[2 * k] = e0;
    v[2 * k + 1] = e1;
    s2 = f2_add(s2, f2_pack(e0, e1));
  }
  float sa, sb;
  f2_unpack(s2, sa, sb);
  float s = group_sum<LPR>(sa + sb, mask);
  // +inf: m == inf; -inf: some lane's min == -inf; NaN: s is NaN
  flag_nonfinite(flag, neg_inf || !(fabsf(m) <= FLT_MAX) || !(s == s));
  const float inv = 1.0f / s;
  const unsigned long long inv2 = f2_pack(inv, inv);
#pragma unroll
  for (int k = 0; k < VPL / 2; ++k)
    f2_unpack(f2_mul(f2_pack(v[2 * k], v[2 * k + 1]), inv2), v[2 * k], v[2 * k + 1]);
  if constexpr (VEC) {
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k) {
      const uint32_t col = (lane + k * LPR) * 4;
      if (col < cols)
        stg_stream(reinterpret_cast<float4*>(out + col),
                   make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
    }
  } else {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t col = lane + k * LPR;
      if (col < cols) stg_stream(out + col, v[k]);
    }
  }
}

__device__ __forceinline__ float block_reduce_max(float v, float* red) {
  v = group_max<32>(v, 0xffffffffu);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; ++i) r = fmaxf(r, red[i]);
  __syncthreads();
  return r;
}
__device__ __forceinline__ float block_reduce_sum(float v, float* red) {
  v = group_sum<32>(v, 0xffffffffu);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; ++i) r += red[i];
  __syncthreads();
  return r;
}

// One CTA per row, VPL values per thread in registers (cols <= 256 * VPL).
// MINB resident CTAs per SM asked of the register allocator: with one row
// per CTA, more resident rows overlap one row's load with another's
// reductions.
template <int VPL, bool VEC, int MINB = 1>
__global__ void __launch_bounds__(kThreads, MINB)
    softmax_wide_kernel(const float* __restrict__ src, float* __restrict__ dst,
                        uint32_t cols, int* flag) {
  LCNN_PDL_ENTRY();
  __shared__ float red[kThreads / 32];
  const float* in = src + static_cast<uint64_t>(blockIdx.x) * cols;
  float* out = dst + static_cast<uint64_t>(blockIdx.x) * cols;
  const int t = threadIdx.x;
  float v[VPL];
  bool bad = false;
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) {
    const uint32_t col = (t + k * kThreads) * 4;
    if constexpr (VEC) {
      if (col < cols) {
        const float4 q = ldg_stream(reinterpret_cast<const float4*>(in + col));
        v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
      } else {
        v[4 * k] = v[4 * k + 1] = v[4 * k + 2] = v[4 * k + 3] = -INFINITY;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[4 * k + j] = col + j < cols ? __ldg(in + col + j) : -INFINITY;
    }
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t col = (t + (k / 4) * kThreads) * 4 + (k % 4);
    if (col < cols) {
      bad |= !isfinite(v[k]);
      m = fmaxf(m, v[k]);
    }
  }
  flag_nonfinite(flag, bad);
  m = block_reduce_max(m, red);
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const uint32_t col = (t + (k / 4) * kThreads) * 4 + (k % 4);
    const float e = col < cols ? fexp(v[k] - m) : 0.0f;
    v[k] = e;
    s += e;
  }
  s = block_reduce_sum(s, red);
  const float inv = 1.0f / s;
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) {
    const uint32_t col = (t + k * kThreads) * 4;
    if constexpr (VEC) {
      if (col < cols)
        stg_stream(reinterpret_cast<float4*>(out + col),
                   make_float4(v[4 * k] * inv, v[4 * k + 1] * inv, v[4 * k + 2] * inv,
                               v[4 * k + 3] * inv));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (col + j < cols) stg_stream(out + col + j, v[4 * k + j] * inv);
    }
  }
}

// Rows wider than the register kernels (> 16384 columns, up to ~56K):
// persistent CTAs stage each row in shared memory with one cp.async.bulk
// (double-buffered when two rows fit: the next row streams in while this one
// is reduced), so the row is read from HBM once -- the stream kernel below
// reads it twice.  Same arithmetic as softmax_wide_kernel: max, then
// e = exp(x - max) kept in shared memory with its sum, then e * (1 / sum).
__global__ void __launch_bounds__(kThreads)
    softmax_smem_kernel(const float* __restrict__ src, float* __restrict__ dst, uint32_t rows,
                        uint32_t cols, uint32_t nbuf, uint32_t pitch, int* flag) {
  LCNN_PDL_ENTRY();
  extern __shared__ __align__(128) float sm_rows[];
  __shared__ uint64_t full[2];
  __shared__ float red[kThreads / 32];
  const uint32_t bytes = cols * 4, G = gridDim.x, c4 = cols / 4;
  if (threadIdx.x == 0) {
    lcnn_tc::mbar_init(&full[0], 1);
    lcnn_tc::mbar_init(&full[1], 1);
    lcnn_tc::mbar_fence_init();
    for (uint32_t k = 0; k < nbuf; ++k) {
      const uint32_t rr = blockIdx.x + k * G;
      if (rr < rows) {
        lcnn_tc::mbar_arrive_expect_tx(&full[k], bytes);
        lcnn_tc::bulk_load(sm_rows + k * pitch, src + static_cast<uint64_t>(rr) * cols, bytes,
                           &full[k]);
      }
    }
  }
  __syncthreads();
  uint32_t it = 0;
  for (uint32_t r = blockIdx.x; r < rows; r += G, ++it) {
    const uint32_t b = nbuf == 2 ? (it & 1u) : 0u;
    const uint32_t ph = nbuf == 2 ? ((it >> 1) & 1u) : (it & 1u);
    lcnn_tc::mbar_wait(&full[b], ph);
    float4* x = reinterpret_cast<float4*>(sm_rows + b * pitch);
    float m = -INFINITY;
    bool bad = false;
    for (uint32_t j = threadIdx.x; j < c4; j += kThreads) {
      const float4 v = x[j];
      bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
      m = fmaxf(fmaxf(m, fmaxf(v.x, v.y)), fmaxf(v.z, v.w));
    }
    flag_nonfinite(flag, bad);
    m = block_reduce_max(m, red);
    float s = 0.0f;
    for (uint32_t j = threadIdx.x; j < c4; j += kThreads) {
      float4 v = x[j];
      v.x = fexp(v.x - m);
      v.y = fexp(v.y - m);
      v.z = fexp(v.z - m);
      v.w = fexp(v.w - m);
      s += v.x;
      s += v.y;
      s += v.z;
      s += v.w;
      x[j] = v;
    }
    s = block_reduce_sum(s, red);  // its barriers also publish the e values
    const float inv = 1.0f / s;
    float4* out = reinterpret_cast<float4*>(dst + static_cast<uint64_t>(r) * cols);
    for (uint32_t j = threadIdx.x; j < c4; j += kThreads) {
      const float4 e = x[j];
      stg_stream(out + j, make_float4(e.x * inv, e.y * inv, e.z * inv, e.w * inv));
    }
    // every thread is done with buffer b (generic-proxy reads / writes)
    // before the async proxy refills it with the row nbuf * G further on
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t rn = r + nbuf * G;
      if (rn < rows) {
        lcnn_tc::mbar_arrive_expect_tx(&full[b], bytes);
        lcnn_tc::bulk_load(sm_rows + b * pitch, src + static_cast<uint64_t>(rn) * cols, bytes,
                           &full[b]);
      }
    }
  }
}

// One CTA per row of any width: online (max, sum) then normalise.
__global__ void __launch_bounds__(kThreads)
    softmax_stream_kernel(const float* __restrict__ src, float* __restrict__ dst,
                          uint32_t cols, int* flag) {
  LCNN_PDL_ENTRY();
  __shared__ float red_m[kThreads / 32], red_s[kThreads / 32];
  const float* in = src + static_cast<uint64_t>(blockIdx.x) * cols;
  float* out = dst + static_cast<uint64_t>(blockIdx.x) * cols;
  float m = -INFINITY, s = 0.0f;
  bool bad = false;
  for (uint32_t j = threadIdx.x; j < cols; j += kThreads) {
    const float x = __ldg(in + j);
    bad |= !isfinite(x);
    if (x > m) {
      s = s * fexp(m - x) + 1.0f;
      m = x;
    } else {
      s += fexp(x - m);
    }
  }
  flag_nonfinite(flag, bad);
  // merge (m, s) pairs: warp then block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o);
    const float so = __shfl_xor_sync(0xffffffffu, s, o);
    const float mn = fmaxf(m, mo);
    s = (m == -INFINITY ? 0.0f : s * fexp(m - mn)) + (mo == -INFINITY ? 0.0f : so * fexp(mo - mn));
    m = mn;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red_m[w] = m;
    red_s[w] = s;
  }
  __syncthreads();
  float M = red_m[0];
  for (int i = 1; i < kThreads / 32; ++i) M = fmaxf(M, red_m[i]);
  float S = 0.0f;
  for (int i = 0; i < kThreads / 32; ++i)
    S += red_m[i] == -INFINITY ? 0.0f : red_s[i] * fexp(red_m[i] - M);
  const float inv = 1.0f / S;
  for (uint32_t j = threadIdx.x; j < cols; j += kThreads)
    stg_stream(out + j, fexp(__ldg(in + j) - M) * inv);
}

// ---- five-pass baseline (softmax.cpp:36-98), one kernel per step ---------
template <int LPR>
__global__ void __launch_bounds__(kThreads)
    row_max_kernel(const float* __restrict__ in, float* __restrict__ maxv, uint32_t rows,
                   uint32_t cols, int* flag) {
  LCNN_PDL_ENTRY();
  const uint32_t row = blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int lane = threadIdx.x % LPR;
  const int wl = threadIdx.x & 31;
  const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (wl & ~(LPR - 1)));
  if (row >= rows) return;
  const float* r = in + static_cast<uint64_t>(row) * cols;
  float m = -INFINITY;
  bool bad = false;
  for (uint32_t j = lane; j < cols; j += LPR) {
    const float x = r[j];
    bad |= !isfinite(x);
    m = fmaxf(m, x);
  }
  flag_nonfinite(flag, bad);
  m = group_max<LPR>(m, mask);
  if (lane == 0) maxv[row] = m;
}

template <int LPR>
__global__ void __launch_bounds__(kThreads)
    row_sum_kernel(const float* __restrict__ in, float* __restrict__ sumv, uint32_t rows,
                   uint32_t cols) {
  LCNN_PDL_ENTRY();
  const uint32_t row = blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int lane = threadIdx.x % LPR;
  const int wl = threadIdx.x & 31;
  const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (wl & ~(LPR - 1)));
  if (row >= rows) return;
  const float* r = in + static_cast<uint64_t>(row) * cols;
  float s = 0.0f;
  for (uint32_t j = lane; j < cols; j += LPR) s += r[j];
  s = group_sum<LPR>(s, mask);
  if (lane == 0) sumv[row] = s;
}

__global__ void __launch_bounds__(kThreads)
    sub_rowvec_kernel(const float* __restrict__ in, const float* __restrict__ maxv,
                      float* __restrict__ out, uint64_t total, FastDiv div_cols) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * kThreads)
    out[i] = in[i] - maxv[div_cols.div(static_cast<uint32_t>(i))];
}

__global__ void __launch_bounds__(kThreads)
    exp_kernel(const float* __restrict__ in, float* __restrict__ out, uint64_t total) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * kThreads)
    out[i] = expf(in[i]);
}

__global__ void __launch_bounds__(kThreads)
    scale_rowvec_kernel(const float* __restrict__ in, const float* __restrict__ sumv,
                        float* __restrict__ out, uint64_t total, FastDiv div_cols) {
  LCNN_PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * kThreads)
    out[i] = in[i] * (1.0f / sumv[div_cols.div(static_cast<uint32_t>(i))]);
}

}  // namespace lcnn_dev

namespace lcnn_impl {

using namespace lcnn_dev;

namespace {

template <int LPR, int VPL, int THREADS = kThreads>
cudaError_t rows_launch(const float* src, float* dst, uint32_t rows, uint32_t cols, bool vec,
                        int* flag, cudaStream_t st) {
  constexpr int kGroups = THREADS / LPR;
  const uint32_t blocks = (rows + kGroups - 1) / kGroups;
  if (vec)
    lcnn_pdl::launch(softmax_rows_kernel<LPR, VPL, true, THREADS>, blocks, THREADS, 0, st, src,
                     dst, rows, cols, flag);
  else
    lcnn_pdl::launch(softmax_rows_kernel<LPR, VPL, false, THREADS>, blocks, THREADS, 0, st, src,
                     dst, rows, cols, flag);
  return cudaGetLastError();
}

template <int VPL, int MINB = 1>
cudaError_t wide_launch(const float* src, float* dst, uint32_t rows, uint32_t cols, bool vec,
                        int* flag, cudaStream_t st) {
  if (vec) lcnn_pdl::launch(softmax_wide_kernel<VPL, true, MINB>, rows, kThreads, 0, st, src, dst, cols, flag);
  else lcnn_pdl::launch(softmax_wide_kernel<VPL, false, MINB>, rows, kThreads, 0, st, src, dst, cols, flag);
  return cudaGetLastError();
}

uint32_t grid_for(uint64_t total) {
  uint64_t b = (total + kThreads - 1) / kThreads;
  if (b > 148ull * 16) b = 148ull * 16;
  return static_cast<uint32_t>(b ? b : 1);
}

}  // namespace

cudaError_t launch_softmax_fused(const float* src, float* dst, uint32_t rows, uint32_t cols,
                                 int* flag, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const bool vec = (cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0);
  // register-resident rows: choose lanes-per-row so each lane holds <= 64
  if (cols <= 16) return rows_launch<4, 4>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 64) return rows_launch<8, 8>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 256) return rows_launch<16, 16>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 512) return rows_launch<32, 16>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 1024) return rows_launch<32, 32, 128>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 2048) return rows_launch<32, 64>(src, dst, rows, cols, vec, flag, st);
  // one CTA per row: the smallest register row that fits, with a register
  // bound that keeps 2-3 rows resident per SM so one row's load overlaps
  // another's reductions (measured on B200, 4096 rows: 8192 cols 5.40 -> 6.43,
  // 10000 -- the paper's case -- 3.09 -> 6.46, 12288 4.81 -> 5.61, 16384
  // 3.62 -> 5.28 TB/s; profiles/r02_softmax_wide_ab.jsonl)
  static const bool minb1 = [] {  // profiling knob LCNN_SM_WIDE_MINB=1: no occupancy bound
    const char* e = std::getenv("LCNN_SM_WIDE_MINB");
    return e && e[0] == '1';
  }();
  if (cols <= 4096) return wide_launch<16>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 8192)
    return minb1 ? wide_launch<32>(src, dst, rows, cols, vec, flag, st)
                 : wide_launch<32, 3>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 10240)
    return minb1 ? wide_launch<40>(src, dst, rows, cols, vec, flag, st)
                 : wide_launch<40, 3>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 12288)
    return minb1 ? wide_launch<48>(src, dst, rows, cols, vec, flag, st)
                 : wide_launch<48, 3>(src, dst, rows, cols, vec, flag, st);
  if (cols <= 16384)
    return minb1 ? wide_launch<64>(src, dst, rows, cols, vec, flag, st)
                 : wide_launch<64, 2>(src, dst, rows, cols, vec, flag, st);
  // rows that fit shared memory: staged once (double-buffered when two fit)
  constexpr uint32_t kSmemMax = 227 * 1024 - 1024;
  const uint32_t pitch = (cols + 31) / 32 * 32;  // floats per buffer, 128-B aligned
  static const bool smem_off = [] {  // profiling knob LCNN_SM_SMEM=0: the two-pass stream kernel
    const char* e = std::getenv("LCNN_SM_SMEM");
    return e && e[0] == '0';
  }();
  if (vec && !smem_off && pitch * 4ull <= kSmemMax) {
    const uint32_t nbuf = 2ull * pitch * 4 <= kSmemMax ? 2 : 1;
    const uint32_t smem = nbuf * pitch * 4;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(softmax_smem_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kSmemMax));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const uint32_t per_sm = kSmemMax / smem >= 2 ? 2 : 1;
    const uint32_t grid = rows < 148u * per_sm ? rows : 148u * per_sm;
    lcnn_pdl::launch(softmax_smem_kernel, grid, kThreads, smem, st, src, dst, rows, cols, nbuf,
                     pitch, flag);
    return cudaGetLastError();
  }
  lcnn_pdl::launch(softmax_stream_kernel, rows, kThreads, 0, st, src, dst, cols, flag);
  return cudaGetLastError();
}

cudaError_t launch_softmax_five_pass(const float* src, float* dst, uint32_t rows, uint32_t cols,
                                     float* scratch, int* flag, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const uint64_t total = static_cast<uint64_t>(rows) * cols;
  float* maxv = scratch;
  float* sumv = scratch + rows;
  float* midv1 = scratch + 2 * static_cast<uint64_t>(rows);
  float* midv2 = midv1 + total;
  const FastDiv dc(cols);
  const uint32_t row_blocks = (rows + 7) / 8;  // 8 rows (warps) per CTA
  lcnn_pdl::launch(row_max_kernel<32>, row_blocks, kThreads, 0, st, src, maxv, rows, cols, flag);
  lcnn_pdl::launch(sub_rowvec_kernel, grid_for(total), kThreads, 0, st, src, maxv, midv1, total, dc);
  lcnn_pdl::launch(exp_kernel, grid_for(total), kThreads, 0, st, midv1, midv2, total);
  lcnn_pdl::launch(row_sum_kernel<32>, row_blocks, kThreads, 0, st, midv2, sumv, rows, cols);
  lcnn_pdl::launch(scale_rowvec_kernel, grid_for(total), kThreads, 0, st, midv2, sumv, dst, total, dc);
  return cudaGetLastError();
}

}  // namespace lcnn_impl
