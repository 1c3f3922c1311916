// Device-side helpers shared by the sm_100a kernels of the layer path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "launch.cuh"

namespace lcnn_dev {

constexpr int kThreads = 256;

// Unsigned 32-bit division by a runtime constant (Granlund-Montgomery):
// q = umulhi(x, mul) >> shift, exact for every 32-bit x.  Index math in the
// kernels runs once per element, so a hardware divide (~20 instructions)
// would cost more issue slots than the memory traffic it serves.
struct FastDiv {
  uint32_t d, mul, shift;
  FastDiv() = default;
  explicit FastDiv(uint32_t divisor) : d(divisor) {
    if (divisor <= 1) {  // x / 1: mul = 0 handled below with shift = 0
      mul = 0;
      shift = 0;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < divisor) ++l;
    shift = l - 1;
    // mul = floor(2^32 * (2^l - d) / d) + 1
    const uint64_t num = (uint64_t{1} << 32) * ((uint64_t{1} << l) - divisor);
    mul = static_cast<uint32_t>(num / divisor + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    if (d == 1) return x;
    const uint32_t t = __umulhi(x, mul);
    return (t + ((x - t) >> 1)) >> shift;
  }
  __device__ __forceinline__ void divmod(uint32_t x, uint32_t& q,
                                         uint32_t& r) const {
    q = div(x);
    r = x - q * d;
  }
};

// std::max(acc, v) from libstdc++ is (acc < v) ? v : acc: NaN taps never
// replace the running value and ties keep the earlier tap (pool.cpp:120,153).
__device__ __forceinline__ float max_tap(float acc, float v) {
  return (acc < v) ? v : acc;
}

__device__ __forceinline__ float4 max_tap(float4 acc, float4 v) {
  return make_float4(max_tap(acc.x, v.x), max_tap(acc.y, v.y),
                     max_tap(acc.z, v.z), max_tap(acc.w, v.w));
}

// Explicit round-to-nearest ops so nvcc can never contract into FMA: the
// average pool must reproduce the reference's fp32 operation sequence.
__device__ __forceinline__ float add_tap(float acc, float v) {
  return __fadd_rn(acc, v);
}
__device__ __forceinline__ float4 add_tap(float4 acc, float4 v) {
  return make_float4(__fadd_rn(acc.x, v.x), __fadd_rn(acc.y, v.y),
                     __fadd_rn(acc.z, v.z), __fadd_rn(acc.w, v.w));
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
  asm volatile("st.global" LCNN_ST_HINT ".v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void stg_stream(float* p, float v) {
  asm volatile("st.global" LCNN_ST_HINT ".f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
};
template <>
struct Vec<4> {
  using T = float4;
};

template <int VEC>
__device__ __forceinline__ typename Vec<VEC>::T splat(float x);
template <>
__device__ __forceinline__ float splat<1>(float x) {
  return x;
}
template <>
__device__ __forceinline__ float4 splat<4>(float x) {
  return make_float4(x, x, x, x);
}

__device__ __forceinline__ float scale_out(float a, float s) {
  return __fmul_rn(a, s);
}
__device__ __forceinline__ float4 scale_out(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s),
                     __fmul_rn(a.w, s));
}
__device__ __forceinline__ float divide_out(float a, float d) {
  return __fdiv_rn(a, d);
}
__device__ __forceinline__ float4 divide_out(float4 a, float d) {
  return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d),
                     __fdiv_rn(a.w, d));
}

}  // namespace lcnn_dev
