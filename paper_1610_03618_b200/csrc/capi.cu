// C ABI (include/lcnn_cuda.h): host-side validation with the reference's
// rules and messages, analytic access/pass reports, kernel dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/lcnn_cuda.h"
#include "internal.h"

namespace {

thread_local std::string g_last_error;

lcnn_status fail(lcnn_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

lcnn_status ok() {
  g_last_error.clear();
  return LCNN_OK;
}

lcnn_status cuda_fail(cudaError_t e, const char* where) {
  return fail(LCNN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

bool valid_layout(int l) { return l >= LCNN_NCHW && l <= LCNN_HWCN; }

// checked_volume (tensor.cpp:16-29)
lcnn_status check_volume(uint32_t n, uint32_t c, uint32_t h, uint32_t w, const char* what) {
  if (n == 0 || c == 0 || h == 0 || w == 0)
    return fail(LCNN_ESHAPE, std::string(what) + ": all dims must be >= 1");
  const uint64_t v = uint64_t{n} * c * uint64_t{h} * w;
  if (v > 0xffffffffull) return fail(LCNN_ESHAPE, std::string(what) + ": dim product overflows");
  return LCNN_OK;
}

bool power_of_two(uint32_t v) { return v != 0 && (v & (v - 1)) == 0; }

// check_window (pool.cpp:19-26)
lcnn_status check_window(uint32_t h, uint32_t w, uint32_t wh, uint32_t ww, uint32_t s) {
  if (wh < 1 || ww < 1 || s < 1) return fail(LCNN_ESHAPE, "pool: window and stride must be >= 1");
  if (wh > h || ww > w) return fail(LCNN_ESHAPE, "pool: window larger than image");
  return LCNN_OK;
}

// covered_extent (pool.cpp:29-33)
uint64_t covered_extent(uint32_t out, uint32_t win, uint32_t stride) {
  if (stride >= win) return uint64_t{out} * win;
  return uint64_t{stride} * (out - 1) + win;
}

void plain_report(lcnn_access_report* r, uint32_t n, uint32_t c, uint32_t ho, uint32_t wo,
                  uint32_t wh, uint32_t ww, uint32_t s) {
  if (!r) return;
  const uint64_t outs = uint64_t{n} * c * ho * wo;
  r->output_stores = outs;
  r->input_loads = outs * wh * ww;
  r->distinct_inputs = uint64_t{n} * c * covered_extent(ho, wh, s) * covered_extent(wo, ww, s);
}

// union-load formula of pool_coarsened (pool.cpp:216-236)
void coarsened_report(lcnn_access_report* r, uint32_t n, uint32_t c, uint32_t ho, uint32_t wo,
                      uint32_t wh, uint32_t ww, uint32_t s, uint32_t fh, uint32_t fw) {
  if (!r) return;
  uint64_t total = 0;
  for (uint32_t oh0 = 0; oh0 < ho; oh0 += fh) {
    const uint32_t bh = (fh < ho - oh0) ? fh : ho - oh0;
    for (uint32_t ow0 = 0; ow0 < wo; ow0 += fw) {
      const uint32_t bw = (fw < wo - ow0) ? fw : wo - ow0;
      total += uint64_t{s * (bh - 1) + wh} * (s * (bw - 1) + ww);
    }
  }
  r->input_loads = total * n * c;
  r->output_stores = uint64_t{n} * c * ho * wo;
  r->distinct_inputs = uint64_t{n} * c * covered_extent(ho, wh, s) * covered_extent(wo, ww, s);
}

lcnn_status pool_common(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                        uint32_t w, uint32_t wh, uint32_t ww, uint32_t s, int mode,
                        uint32_t* ho, uint32_t* wo) {
  if (!src || !dst) return fail(LCNN_EINVAL, "pool: null tensor pointer");
  if (mode != LCNN_POOL_MAX && mode != LCNN_POOL_AVG) return fail(LCNN_EINVAL, "pool: bad mode");
  lcnn_status st = check_volume(n, c, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  st = check_window(h, w, wh, ww, s);
  if (st != LCNN_OK) return st;
  *ho = (h - wh) / s + 1;  // pool_output_extents (pool.cpp:44-47)
  *wo = (w - ww) / s + 1;
  return LCNN_OK;
}

}  // namespace

extern "C" {

int lcnn_abi_version(void) { return LCNN_ABI_VERSION; }

const char* lcnn_last_error(void) { return g_last_error.c_str(); }

const char* lcnn_status_name(int status) {
  switch (status) {
    case LCNN_OK: return "ok";
    case LCNN_ESHAPE: return "ShapeError";
    case LCNN_EINDEX: return "IndexError";
    case LCNN_ELAYOUT: return "LayoutError";
    case LCNN_EPLAN: return "PlanError";
    case LCNN_EFORMAT: return "FormatError";
    case LCNN_EDOMAIN: return "DomainError";
    case LCNN_EUNSUPPORTED: return "UnsupportedError";
    case LCNN_EVALIDATION: return "ValidationError";
    case LCNN_ECALIBRATION: return "CalibrationError";
    case LCNN_ECUDA: return "CudaError";
    case LCNN_EINVAL: return "InvalidArgument";
    default: return "unknown";
  }
}

int lcnn_device_ok(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
    return 0;
  return major == 10 ? 1 : 0;
}

int lcnn_flattenable_pair(int src, int dst) {
  return (src == LCNN_CHWN && dst == LCNN_NCHW) || (src == LCNN_NCHW && dst == LCNN_CHWN);
}

lcnn_status lcnn_transform_naive(const float* src, float* dst, uint32_t n, uint32_t c,
                                 uint32_t h, uint32_t w, int src_layout, int dst_layout,
                                 void* stream) {
  if (!src || !dst) return fail(LCNN_EINVAL, "transform: null tensor pointer");
  if (!valid_layout(src_layout) || !valid_layout(dst_layout))
    return fail(LCNN_EINVAL, "transform: bad layout code");
  lcnn_status st = check_volume(n, c, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  cudaError_t e = lcnn_impl::launch_permute4d(src, dst, n, c, h, w, src_layout, dst_layout,
                                              S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "transform_naive");
  return ok();
}

lcnn_status lcnn_transform_tiled(const float* src, float* dst, uint32_t n, uint32_t c,
                                 uint32_t h, uint32_t w, int src_layout, int dst_layout,
                                 uint32_t tile, int wide_copy, void* stream) {
  if (!src || !dst) return fail(LCNN_EINVAL, "transform: null tensor pointer");
  if (!valid_layout(src_layout) || !valid_layout(dst_layout))
    return fail(LCNN_EINVAL, "transform: bad layout code");
  lcnn_status st = check_volume(n, c, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  // validate_plan (layout.cpp:13-26)
  if (!lcnn_flattenable_pair(src_layout, dst_layout))
    return fail(LCNN_EPLAN,
                "transform_tiled: unsupported layout pair (only CHWN<->NCHW flattens)");
  if (!power_of_two(tile) || tile < 8 || tile > 128)
    return fail(LCNN_EPLAN, "transform_tiled: tile must be a power of two in [8, 128]");
  if (wide_copy && n < 64) return fail(LCNN_EPLAN, "transform_tiled: wide copy requires N >= 64");
  const uint64_t flat = uint64_t{c} * h * w;
  // CHWN: [CHW][N] -> [N][CHW];  NCHW: [N][CHW] -> [CHW][N]
  const uint64_t rows = src_layout == LCNN_CHWN ? flat : n;
  const uint64_t cols = src_layout == LCNN_CHWN ? n : flat;
  cudaError_t e = lcnn_impl::launch_transpose2d(src, dst, rows, cols, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "transform_tiled");
  return ok();
}

lcnn_status lcnn_transform(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                           uint32_t w, int src_layout, int dst_layout, void* stream) {
  if (!src || !dst) return fail(LCNN_EINVAL, "transform: null tensor pointer");
  if (!valid_layout(src_layout) || !valid_layout(dst_layout))
    return fail(LCNN_EINVAL, "transform: bad layout code");
  // make_plan (layout.cpp:122-136) + dispatch (layout.cpp:138-144)
  if (lcnn_flattenable_pair(src_layout, dst_layout))
    return lcnn_transform_tiled(src, dst, n, c, h, w, src_layout, dst_layout, 32, n >= 64, stream);
  if (src_layout == dst_layout) {
    lcnn_status st = check_volume(n, c, h, w, "Tensor4D");
    if (st != LCNN_OK) return st;
    cudaError_t e = cudaMemcpyAsync(dst, src, uint64_t{n} * c * h * w * sizeof(float),
                                    cudaMemcpyDeviceToDevice, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "transform");
    return ok();
  }
  return lcnn_transform_naive(src, dst, n, c, h, w, src_layout, dst_layout, stream);
}

lcnn_status lcnn_pool_output_extents(uint32_t h, uint32_t w, uint32_t win_h, uint32_t win_w,
                                     uint32_t stride, uint32_t* h_out, uint32_t* w_out) {
  if (!h_out || !w_out) return fail(LCNN_EINVAL, "pool: null output pointer");
  lcnn_status st = check_window(h, w, win_h, win_w, stride);
  if (st != LCNN_OK) return st;
  *h_out = (h - win_h) / stride + 1;
  *w_out = (w - win_w) / stride + 1;
  return ok();
}

// ---- pooling plans: static defaults, the GPU tuner and its cache ---------
namespace {

// The plan pool_layout uses before (or without) tuning.  NCHW: the pipelined
// kernel's output block measured in round 1 (scripts/pool_plans.py,
// profiles/r01_pool_plans_nchw*.txt: 3x3/s2 -> 3x2; 2x2/s2 -> 2x2 on >= 200-wide
// planes, 4x1 >= 100, 2x1 >= 20, else 1x2).  CHWN: the plain kernel (1,1).
lcnn_pool_plan static_plan(uint32_t w, int layout, uint32_t win_h, uint32_t win_w,
                           uint32_t stride) {
  lcnn_pool_plan p{1, 1, 0, 0, 0, 0, 0.0f};
  if (layout == LCNN_NCHW && win_h == win_w && stride == 2 && win_h == 3) {
    p.fh = 3;
    p.fw = 2;
  } else if (layout == LCNN_NCHW && win_h == win_w && stride == 2 && win_h == 2) {
    p.fh = w >= 200 ? 2 : w >= 100 ? 4 : w >= 20 ? 2 : 1;
    p.fw = w >= 200 ? 2 : w >= 20 ? 1 : 2;
  }
  return p;
}

using PlanKey = std::tuple<int, uint32_t, uint32_t, uint32_t, uint32_t, int, uint32_t, uint32_t,
                           uint32_t, int>;
std::mutex g_plan_mu;
std::map<PlanKey, lcnn_pool_plan> g_plans;

PlanKey plan_key(uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout, uint32_t win_h,
                 uint32_t win_w, uint32_t stride, int mode) {
  int dev = 0;
  cudaGetDevice(&dev);
  return PlanKey{dev, n, c, h, w, layout, win_h, win_w, stride, mode};
}

lcnn_impl::PoolArgs plan_args(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                              uint32_t w, uint32_t ho, uint32_t wo, uint32_t win_h,
                              uint32_t win_w, uint32_t stride, int mode,
                              const lcnn_pool_plan& p) {
  lcnn_impl::PoolArgs a{src, dst, n, c, h, w, ho, wo, win_h, win_w, stride,
                        mode == LCNN_POOL_AVG, p.fh, p.fw};
  a.ring_kb = p.ring_kb;
  a.ring_slots = p.ring_slots;
  a.ring_ctas = p.ring_ctas;
  return a;
}

cudaError_t launch_plan(const lcnn_impl::PoolArgs& a, int layout, cudaStream_t st) {
  return layout == LCNN_CHWN ? lcnn_impl::launch_pool_chwn(a, st)
                             : lcnn_impl::launch_pool_nchw(a, st);
}

}  // namespace

lcnn_status lcnn_pool_plan_lookup(uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout,
                                  uint32_t win_h, uint32_t win_w, uint32_t stride, int mode,
                                  lcnn_pool_plan* plan) {
  if (!plan) return fail(LCNN_EINVAL, "pool_plan: null plan pointer");
  lcnn_status st = check_window(h, w, win_h, win_w, stride);
  if (st != LCNN_OK) return st;
  if (layout != LCNN_CHWN && layout != LCNN_NCHW)
    return fail(LCNN_ELAYOUT, "pool_layout: only CHWN and NCHW kernels exist");
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    const auto it = g_plans.find(plan_key(n, c, h, w, layout, win_h, win_w, stride, mode));
    if (it != g_plans.end()) {
      *plan = it->second;
      return ok();
    }
  }
  *plan = static_plan(w, layout, win_h, win_w, stride);
  return ok();
}

lcnn_status lcnn_pool_tune(uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout,
                           uint32_t win_h, uint32_t win_w, uint32_t stride, int mode,
                           lcnn_pool_plan* plan, void* stream) {
  lcnn_status st = lcnn_pool_plan_lookup(n, c, h, w, layout, win_h, win_w, stride, mode, plan);
  if (st != LCNN_OK || plan->tuned) return st;
  st = check_volume(n, c, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  if (mode != LCNN_POOL_MAX && mode != LCNN_POOL_AVG) return fail(LCNN_EINVAL, "pool: bad mode");
  const uint32_t ho = (h - win_h) / stride + 1, wo = (w - win_w) / stride + 1;
  const size_t in_bytes = size_t{n} * c * h * w * 4, out_bytes = size_t{n} * c * ho * wo * 4;
  cudaStream_t s = S(stream);
  float *src = nullptr, *dst = nullptr;
  cudaError_t e = cudaMallocAsync(&src, in_bytes, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dst, out_bytes, s);
  // the timing of max / average pooling does not depend on the values
  if (e == cudaSuccess) e = cudaMemsetAsync(src, 0x3f, in_bytes, s);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  if (e != cudaSuccess) {
    if (src) cudaFreeAsync(src, s);
    if (dst) cudaFreeAsync(dst, s);
    return cuda_fail(e, "pool_tune");
  }
  // A layer too big to stay in L2 between layers (in + out > 96 MB) is timed
  // DRAM-cold, as it runs: a 256 MB scratch write evicts L2 before every
  // timed launch (repeated launches on one buffer otherwise hit L2 in part,
  // and ranked the NCHW ring shapes of PL5 differently from a cold run).
  void* flush = nullptr;
  constexpr size_t kFlushBytes = size_t{256} << 20;
  if (in_bytes + out_bytes > (size_t{96} << 20) && cudaMallocAsync(&flush, kFlushBytes, s) != cudaSuccess) {
    cudaGetLastError();
    flush = nullptr;
  }
  // median of `reps` timed launches after one warm-up; a candidate whose
  // launch fails (no specialisation, shared memory over the limit) is skipped
  auto cost = [&](const lcnn_pool_plan& p, int reps = 3) -> float {
    const lcnn_impl::PoolArgs a =
        plan_args(src, dst, n, c, h, w, ho, wo, win_h, win_w, stride, mode, p);
    if (launch_plan(a, layout, s) != cudaSuccess) {
      cudaGetLastError();
      return -1.0f;
    }
    float t[9];
    for (int i = 0; i < reps; ++i) {
      if (flush) cudaMemsetAsync(flush, i, kFlushBytes, s);
      cudaEventRecord(e0, s);
      launch_plan(a, layout, s);
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess) {
        cudaGetLastError();
        return -1.0f;
      }
      cudaEventElapsedTime(&t[i], e0, e1);
    }
    std::sort(t, t + reps);
    return t[reps / 2] * 1e3f;
  };
  // every candidate's screening cost is kept; the closest ones are re-timed
  // with 9 launches at the end (3-launch medians of plans within a few
  // percent of each other picked different winners on different boxes)
  std::vector<lcnn_pool_plan> seen;
  lcnn_pool_plan best = static_plan(w, layout, win_h, win_w, stride);
  best.us = cost(best);
  if (best.us > 0.0f) seen.push_back(best);
  auto consider = [&](lcnn_pool_plan p) {
    const float us = cost(p);
    if (us > 0.0f) {
      p.us = us;
      seen.push_back(p);
    }
    if (us > 0.0f && (best.us <= 0.0f || us < best.us)) best = p;
  };
  // output blocks: every specialised (fh, fw) of the layout's kernel family
  const uint32_t fw_max = layout == LCNN_CHWN ? 4 : 2;
  const bool special = win_h == win_w && ((stride == 2 && (win_h == 2 || win_h == 3)) ||
                                          (stride == 1 && win_h == 3));
  if (special)
    for (uint32_t fh = 1; fh <= 4; ++fh)
      for (uint32_t fw = 1; fw <= fw_max; ++fw)
        if (fh != best.fh || fw != best.fw) consider(lcnn_pool_plan{fh, fw, 0, 0, 0, 0, 0.0f});
  // NCHW pipelined kernel: the shared-memory ring for the chosen block
  // (KB per slot, slots, CTAs per SM); ineligible shapes ignore the ring
  if (layout == LCNN_NCHW && special) {
    static const uint32_t rings[][3] = {{48, 2, 2}, {24, 2, 4}, {32, 2, 3}, {16, 3, 4},
                                        {24, 3, 3}, {64, 2, 1}, {12, 4, 4}};
    const lcnn_pool_plan base = best;
    for (const auto& r : rings) {
      lcnn_pool_plan p = base;
      p.ring_kb = r[0];
      p.ring_slots = r[1];
      p.ring_ctas = r[2];
      consider(p);
    }
  }
  // refine: the candidates within 5 % of the screening winner, 9 launches each
  if (best.us > 0.0f) {
    const float cut = best.us * 1.05f;
    lcnn_pool_plan win = best;
    win.us = -1.0f;
    for (lcnn_pool_plan p : seen) {
      if (p.us > cut) continue;
      const float us = cost(p, 9);
      if (us > 0.0f && (win.us <= 0.0f || us < win.us)) {
        p.us = us;
        win = p;
      }
    }
    if (win.us > 0.0f) best = win;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(src, s);
  cudaFreeAsync(dst, s);
  if (flush) cudaFreeAsync(flush, s);
  cudaGetLastError();
  if (best.us <= 0.0f) return fail(LCNN_ECUDA, "pool_tune: no candidate launched");
  best.tuned = 1;
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    g_plans[plan_key(n, c, h, w, layout, win_h, win_w, stride, mode)] = best;
  }
  *plan = best;
  return ok();
}

lcnn_status lcnn_pool_run_plan(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                               uint32_t w, int layout, uint32_t win_h, uint32_t win_w,
                               uint32_t stride, int mode, const lcnn_pool_plan* plan,
                               lcnn_access_report* report, void* stream) {
  uint32_t ho = 0, wo = 0;
  lcnn_status st = pool_common(src, dst, n, c, h, w, win_h, win_w, stride, mode, &ho, &wo);
  if (st != LCNN_OK) return st;
  if (layout != LCNN_CHWN && layout != LCNN_NCHW)
    return fail(LCNN_ELAYOUT, "pool_layout: only CHWN and NCHW kernels exist");
  if (!plan) return fail(LCNN_EINVAL, "pool_plan: null plan pointer");
  if (plan->fh < 1 || plan->fw < 1) return fail(LCNN_EPLAN, "pool_coarsened: factors must be >= 1");
  if (uint64_t{plan->fh} * plan->fw > 64)
    return fail(LCNN_EPLAN, "pool_coarsened: fh*fw exceeds accumulator cap of 64");
  const lcnn_impl::PoolArgs a =
      plan_args(src, dst, n, c, h, w, ho, wo, win_h, win_w, stride, mode, *plan);
  cudaError_t e = launch_plan(a, layout, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pool_run_plan");
  coarsened_report(report, n, c, ho, wo, win_h, win_w, stride, plan->fh, plan->fw);
  return ok();
}

lcnn_status lcnn_pool_layout(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                             uint32_t w, int layout, uint32_t win_h, uint32_t win_w,
                             uint32_t stride, int mode, lcnn_access_report* report,
                             void* stream) {
  uint32_t ho = 0, wo = 0;
  lcnn_status st = pool_common(src, dst, n, c, h, w, win_h, win_w, stride, mode, &ho, &wo);
  if (st != LCNN_OK) return st;
  if (layout != LCNN_CHWN && layout != LCNN_NCHW)
    return fail(LCNN_ELAYOUT, "pool_layout: only CHWN and NCHW kernels exist");
  // the tuned plan of this shape if lcnn_pool_tune has measured it, else the
  // static default.  Every output keeps its tap order under any plan, so the
  // bits equal the plain kernel's and the report stays the plain one.
  lcnn_pool_plan p;
  st = lcnn_pool_plan_lookup(n, c, h, w, layout, win_h, win_w, stride, mode, &p);
  if (st != LCNN_OK) return st;
  const lcnn_impl::PoolArgs a = plan_args(src, dst, n, c, h, w, ho, wo, win_h, win_w, stride,
                                          mode, p);
  cudaError_t e = launch_plan(a, layout, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pool_layout");
  plain_report(report, n, c, ho, wo, win_h, win_w, stride);
  return ok();
}

lcnn_status lcnn_pool_coarsened(const float* src, float* dst, uint32_t n, uint32_t c,
                                uint32_t h, uint32_t w, int layout, uint32_t win_h,
                                uint32_t win_w, uint32_t stride, int mode, uint32_t fh,
                                uint32_t fw, lcnn_access_report* report, void* stream) {
  uint32_t ho = 0, wo = 0;
  lcnn_status st = pool_common(src, dst, n, c, h, w, win_h, win_w, stride, mode, &ho, &wo);
  if (st != LCNN_OK) return st;
  // pool.cpp:182-191, same order as the reference
  if (fh < 1 || fw < 1) return fail(LCNN_EPLAN, "pool_coarsened: factors must be >= 1");
  if (uint64_t{fh} * fw > 64)
    return fail(LCNN_EPLAN, "pool_coarsened: fh*fw exceeds accumulator cap of 64");
  if (layout != LCNN_CHWN) return fail(LCNN_ELAYOUT, "pool_coarsened: input must be CHWN");
  lcnn_impl::PoolArgs a{src, dst, n, c, h, w, ho, wo, win_h, win_w, stride,
                        mode == LCNN_POOL_AVG, fh, fw};
  cudaError_t e = lcnn_impl::launch_pool_chwn(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pool_coarsened");
  coarsened_report(report, n, c, ho, wo, win_h, win_w, stride, fh, fw);
  return ok();
}

lcnn_status lcnn_pool_coarsened_nchw(const float* src, float* dst, uint32_t n, uint32_t c,
                                     uint32_t h, uint32_t w, uint32_t win_h, uint32_t win_w,
                                     uint32_t stride, int mode, uint32_t fh, uint32_t fw,
                                     lcnn_access_report* report, void* stream) {
  uint32_t ho = 0, wo = 0;
  lcnn_status st = pool_common(src, dst, n, c, h, w, win_h, win_w, stride, mode, &ho, &wo);
  if (st != LCNN_OK) return st;
  if (fh < 1 || fw < 1) return fail(LCNN_EPLAN, "pool_coarsened: factors must be >= 1");
  if (uint64_t{fh} * fw > 64)
    return fail(LCNN_EPLAN, "pool_coarsened: fh*fw exceeds accumulator cap of 64");
  lcnn_impl::PoolArgs a{src, dst, n, c, h, w, ho, wo, win_h, win_w, stride,
                        mode == LCNN_POOL_AVG, fh, fw};
  cudaError_t e = lcnn_impl::launch_pool_nchw(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pool_coarsened_nchw");
  coarsened_report(report, n, c, ho, wo, win_h, win_w, stride, fh, fw);
  return ok();
}

lcnn_status lcnn_pool_oracle(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                             uint32_t w, int layout, uint32_t win_h, uint32_t win_w,
                             uint32_t stride, int mode, void* stream) {
  uint32_t ho = 0, wo = 0;
  lcnn_status st = pool_common(src, dst, n, c, h, w, win_h, win_w, stride, mode, &ho, &wo);
  if (st != LCNN_OK) return st;
  if (!valid_layout(layout)) return fail(LCNN_EINVAL, "pool_oracle: bad layout code");
  // layout_strides (tensor.cpp:55-85)
  uint64_t sn, sc, sh, sw;
  switch (layout) {
    case LCNN_NCHW: sw = 1; sh = w; sc = uint64_t{h} * w; sn = uint64_t{c} * h * w; break;
    case LCNN_CHWN: sn = 1; sw = n; sh = uint64_t{w} * n; sc = uint64_t{h} * w * n; break;
    case LCNN_NHWC: sc = 1; sw = c; sh = uint64_t{w} * c; sn = uint64_t{h} * w * c; break;
    default: sn = 1; sc = n; sw = uint64_t{c} * n; sh = uint64_t{w} * c * n; break;
  }
  lcnn_impl::PoolArgs a{src, dst, n, c, h, w, ho, wo, win_h, win_w, stride,
                        mode == LCNN_POOL_AVG, 1, 1};
  cudaError_t e = lcnn_impl::launch_pool_oracle(a, sn, sc, sh, sw, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pool_oracle");
  return ok();
}

lcnn_status lcnn_softmax_fused(const float* src, float* dst, uint32_t rows, uint32_t cols,
                               uint32_t local_buffer_limit, int* d_nonfinite,
                               lcnn_pass_report* report, void* stream) {
  if (rows < 1 || cols < 1) return fail(LCNN_ESHAPE, "softmax: empty matrix");
  if (!src || !dst) return fail(LCNN_EINVAL, "softmax: null matrix pointer");
  if (uint64_t{rows} * cols > 0xffffffffull)
    return fail(LCNN_ESHAPE, "softmax: matrix too large");
  cudaError_t e = cudaSuccess;
  if (d_nonfinite) {
    e = lcnn_impl::launch_zero2d(d_nonfinite, 1, 1, 1, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "softmax_fused");
  }
  e = lcnn_impl::launch_softmax_fused(src, dst, rows, cols, d_nonfinite, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "softmax_fused");
  if (report) {  // softmax.cpp:142, 178
    report->materializations = 0;
    report->full_matrix_sweeps = cols <= local_buffer_limit ? 2 : 5;
  }
  return ok();
}

lcnn_status lcnn_softmax_fused_sticky(const float* src, float* dst, uint32_t rows, uint32_t cols,
                                      int* d_sticky, void* stream) {
  if (rows < 1 || cols < 1) return fail(LCNN_ESHAPE, "softmax: empty matrix");
  if (!src || !dst) return fail(LCNN_EINVAL, "softmax: null matrix pointer");
  if (uint64_t{rows} * cols > 0xffffffffull)
    return fail(LCNN_ESHAPE, "softmax: matrix too large");
  cudaError_t e = lcnn_impl::launch_softmax_fused(src, dst, rows, cols, d_sticky, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "softmax_fused");
  return ok();
}

size_t lcnn_softmax_reference_scratch_bytes(uint32_t rows, uint32_t cols) {
  return (2 * uint64_t{rows} + 2 * uint64_t{rows} * cols) * sizeof(float);
}

lcnn_status lcnn_softmax_reference(const float* src, float* dst, uint32_t rows, uint32_t cols,
                                   void* d_scratch, size_t scratch_bytes, int* d_nonfinite,
                                   lcnn_pass_report* report, void* stream) {
  if (rows < 1 || cols < 1) return fail(LCNN_ESHAPE, "softmax: empty matrix");
  if (!src || !dst || !d_scratch) return fail(LCNN_EINVAL, "softmax: null pointer");
  if (uint64_t{rows} * cols > 0xffffffffull)
    return fail(LCNN_ESHAPE, "softmax: matrix too large");
  if (scratch_bytes < lcnn_softmax_reference_scratch_bytes(rows, cols))
    return fail(LCNN_EINVAL, "softmax_reference: scratch too small");
  cudaError_t e = cudaSuccess;
  if (d_nonfinite) {
    e = lcnn_impl::launch_zero2d(d_nonfinite, 1, 1, 1, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "softmax_reference");
  }
  e = lcnn_impl::launch_softmax_five_pass(src, dst, rows, cols, static_cast<float*>(d_scratch),
                                          d_nonfinite, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "softmax_reference");
  if (report) {  // softmax.cpp:61-94
    report->materializations = 3;
    report->full_matrix_sweeps = 8;
  }
  return ok();
}

lcnn_status lcnn_conv_output_extents(uint32_t h, uint32_t w, uint32_t f_h, uint32_t f_w,
                                     uint32_t stride, uint32_t pad, uint32_t* h_out,
                                     uint32_t* w_out) {
  if (!h_out || !w_out) return fail(LCNN_EINVAL, "conv: null output pointer");
  if (stride < 1) return fail(LCNN_ESHAPE, "conv: stride must be >= 1");  // conv.cpp:25
  const int64_t span_h = int64_t{h} + 2 * int64_t{pad} - f_h;
  const int64_t span_w = int64_t{w} + 2 * int64_t{pad} - f_w;
  if (span_h < 0 || span_w < 0) return fail(LCNN_ESHAPE, "conv: window larger than padded input");
  *h_out = static_cast<uint32_t>(span_h / stride + 1);
  *w_out = static_cast<uint32_t>(span_w / stride + 1);
  return ok();
}

size_t lcnn_conv_workspace_bytes_ex(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                                    uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                                    uint32_t pad, int precision) {
  if (!stride || f_h > h + 2 * pad || f_w > w + 2 * pad) return 0;
  const uint32_t ho = (h + 2 * pad - f_h) / stride + 1, wo = (w + 2 * pad - f_w) / stride + 1;
  lcnn_impl::ConvArgs a{nullptr, nullptr, nullptr, n, c_i, h, w, c_o, f_h, f_w, stride, pad, ho,
                        wo, layout, precision, nullptr};
  return lcnn_impl::conv_workspace_bytes(a);
}

size_t lcnn_conv_workspace_bytes(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, uint32_t c_o,
                                 uint32_t f_h, uint32_t f_w, int precision) {
  // No stride / padding in this query, and the route (SHARE / ROW / CI / WIN,
  // TAPS-N) depends on both: return the largest need over both layouts, every
  // stride up to the filter size (and 2x beyond) and every padding below the
  // filter size, so the bound holds for whatever geometry the call uses.
  size_t best = 0;
  const uint32_t fmax = f_h > f_w ? f_h : f_w;
  for (int layout : {LCNN_CHWN, LCNN_NCHW})
    for (uint32_t stride = 1; stride <= 2 * fmax; ++stride)
      for (uint32_t pad = 0; pad < fmax; ++pad)
        best = std::max(best, lcnn_conv_workspace_bytes_ex(n, c_i, h, w, layout, c_o, f_h, f_w,
                                                           stride, pad, precision));
  return best;
}

namespace {

// Shared validation of the conv entry points; fills a (pointers left null).
lcnn_status conv_args(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout, uint32_t c_o,
                      uint32_t f_h, uint32_t f_w, uint32_t stride, uint32_t pad, int precision,
                      lcnn_impl::ConvArgs* a) {
  if (precision < LCNN_PREC_TF32 || precision > LCNN_PREC_FP32)
    return fail(LCNN_EINVAL, "conv: bad precision");
  lcnn_status st = check_volume(n, c_i, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  st = check_volume(c_o, c_i, f_h, f_w, "FilterBank");
  if (st != LCNN_OK) return st;
  uint32_t ho = 0, wo = 0;
  st = lcnn_conv_output_extents(h, w, f_h, f_w, stride, pad, &ho, &wo);
  if (st != LCNN_OK) return st;
  if (layout != LCNN_CHWN && layout != LCNN_NCHW)
    return fail(LCNN_ELAYOUT, "conv_direct: only CHWN and NCHW kernels exist");  // conv.cpp:211
  *a = lcnn_impl::ConvArgs{nullptr, nullptr, nullptr, n, c_i, h, w, c_o, f_h, f_w, stride, pad,
                           ho, wo, layout, precision, nullptr};
  return LCNN_OK;
}

}  // namespace

lcnn_status lcnn_conv_forward(const float* src, const float* filters, float* dst, uint32_t n,
                              uint32_t c_i, uint32_t h, uint32_t w, int layout, uint32_t c_o,
                              uint32_t f_h, uint32_t f_w, uint32_t stride, uint32_t pad,
                              int precision, void* d_workspace, size_t workspace_bytes,
                              void* stream) {
  if (!src || !filters || !dst) return fail(LCNN_EINVAL, "conv: null pointer");
  lcnn_impl::ConvArgs a;
  lcnn_status st = conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a);
  if (st != LCNN_OK) return st;
  if (workspace_bytes < lcnn_impl::conv_workspace_bytes(a) || (!d_workspace && workspace_bytes))
    return fail(LCNN_EINVAL, "conv: workspace too small");
  a.src = src;
  a.filters = filters;
  a.dst = dst;
  a.workspace = d_workspace;
  cudaError_t e = lcnn_impl::launch_conv(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "conv_forward");
  return ok();
}

size_t lcnn_conv_packed_bytes(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                              uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                              uint32_t pad, int precision) {
  lcnn_impl::ConvArgs a;
  if (conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a) != LCNN_OK)
    return 0;
  return lcnn_impl::conv_packed_bytes(a);
}

size_t lcnn_conv_packed_workspace_bytes(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                        int layout, uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                        uint32_t stride, uint32_t pad, int precision) {
  lcnn_impl::ConvArgs a;
  if (conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a) != LCNN_OK)
    return 0;
  return lcnn_impl::conv_workspace_bytes(a) - lcnn_impl::conv_packed_bytes(a);
}

lcnn_status lcnn_conv_pack_filters(const float* filters, void* d_packed, size_t packed_bytes,
                                   uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                                   uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                                   uint32_t pad, int precision, void* stream) {
  if (!filters || !d_packed) return fail(LCNN_EINVAL, "conv: null pointer");
  if (reinterpret_cast<uintptr_t>(d_packed) & 255u)
    return fail(LCNN_EINVAL, "conv: packed filters must be 256-byte aligned");
  lcnn_impl::ConvArgs a;
  lcnn_status st = conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a);
  if (st != LCNN_OK) return st;
  if (packed_bytes < lcnn_impl::conv_packed_bytes(a))
    return fail(LCNN_EINVAL, "conv: packed buffer too small");
  a.filters = filters;
  cudaError_t e = lcnn_impl::launch_conv_pack(a, d_packed, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "conv_pack_filters");
  return ok();
}

lcnn_status lcnn_conv_forward_packed(const float* src, const void* d_packed, float* dst,
                                     uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                                     uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                                     uint32_t pad, int precision, void* d_workspace,
                                     size_t workspace_bytes, void* stream) {
  return lcnn_conv_forward_packed_ex(src, d_packed, dst, n, c_i, h, w, layout, c_o, f_h, f_w,
                                     stride, pad, precision, d_workspace, workspace_bytes, nullptr,
                                     stream);
}

lcnn_status lcnn_conv_forward_packed_ex(const float* src, const void* d_packed, float* dst,
                                        uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                        int layout, uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                        uint32_t stride, uint32_t pad, int precision,
                                        void* d_workspace, size_t workspace_bytes, void* d_sync,
                                        void* stream) {
  return lcnn_conv_forward_packed_blk(src, d_packed, dst, n, c_i, h, w, layout, c_o, f_h, f_w,
                                      stride, pad, precision, d_workspace, workspace_bytes,
                                      d_sync, 0u, stream);
}

lcnn_status lcnn_conv_forward_packed_blk(const float* src, const void* d_packed, float* dst,
                                         uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                         int layout, uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                         uint32_t stride, uint32_t pad, int precision,
                                         void* d_workspace, size_t workspace_bytes, void* d_sync,
                                         uint32_t flags, void* stream) {
  if (!src || !d_packed || !dst) return fail(LCNN_EINVAL, "conv: null pointer");
  if (reinterpret_cast<uintptr_t>(d_sync) & 7u)
    return fail(LCNN_EINVAL, "conv: sync word must be 8-byte aligned");
  if (reinterpret_cast<uintptr_t>(d_packed) & 255u)
    return fail(LCNN_EINVAL, "conv: packed filters must be 256-byte aligned");
  lcnn_impl::ConvArgs a;
  lcnn_status st = conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a);
  if (st != LCNN_OK) return st;
  const size_t need = lcnn_impl::conv_workspace_bytes(a) - lcnn_impl::conv_packed_bytes(a);
  if (workspace_bytes < need || (!d_workspace && workspace_bytes))
    return fail(LCNN_EINVAL, "conv: workspace too small");
  a.src = src;
  a.dst = dst;
  a.workspace = d_workspace;
  a.zsync = static_cast<unsigned long long*>(d_sync);
  a.blk = flags;
  if (flags && !lcnn_impl::conv_hwcn32_ok(a, 0, 0))
    return fail(LCNN_EUNSUPPORTED, "conv: blocked activation layout not covered by this route");
  cudaError_t e = lcnn_impl::launch_conv_packed(a, d_packed, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "conv_forward_packed");
  return ok();
}

int lcnn_conv_maxpool_supported(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                                uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                                uint32_t pad, int precision, uint32_t pool_win,
                                uint32_t pool_stride) {
  lcnn_impl::ConvArgs a;
  if (conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a) != LCNN_OK)
    return 0;
  return lcnn_impl::conv_maxpool_fusable(a, pool_win, pool_stride) ? 1 : 0;
}

lcnn_status lcnn_conv_maxpool_packed(const float* src, const void* d_packed, float* dst,
                                     uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, int layout,
                                     uint32_t c_o, uint32_t f_h, uint32_t f_w, uint32_t stride,
                                     uint32_t pad, int precision, uint32_t pool_win,
                                     uint32_t pool_stride, void* stream) {
  return lcnn_conv_maxpool_packed_blk(src, d_packed, dst, n, c_i, h, w, layout, c_o, f_h, f_w,
                                      stride, pad, precision, pool_win, pool_stride, 0u, stream);
}

int lcnn_conv_hwcn32_supported(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w, uint32_t c_o,
                               uint32_t f_h, uint32_t f_w, uint32_t stride, uint32_t pad,
                               int precision, uint32_t pool_win, uint32_t pool_stride,
                               uint32_t flags) {
  lcnn_impl::ConvArgs a;
  if (conv_args(n, c_i, h, w, LCNN_CHWN, c_o, f_h, f_w, stride, pad, precision, &a) != LCNN_OK)
    return 0;
  a.blk = flags;
  return lcnn_impl::conv_hwcn32_ok(a, pool_win, pool_stride) ? 1 : 0;
}

lcnn_status lcnn_conv_maxpool_packed_blk(const float* src, const void* d_packed, float* dst,
                                         uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                         int layout, uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                         uint32_t stride, uint32_t pad, int precision,
                                         uint32_t pool_win, uint32_t pool_stride, uint32_t flags,
                                         void* stream) {
  if (!src || !d_packed || !dst) return fail(LCNN_EINVAL, "conv_maxpool: null pointer");
  if (reinterpret_cast<uintptr_t>(d_packed) & 255u)
    return fail(LCNN_EINVAL, "conv_maxpool: packed filters must be 256-byte aligned");
  lcnn_impl::ConvArgs a;
  lcnn_status st = conv_args(n, c_i, h, w, layout, c_o, f_h, f_w, stride, pad, precision, &a);
  if (st != LCNN_OK) return st;
  if (!lcnn_impl::conv_maxpool_fusable(a, pool_win, pool_stride))
    return fail(LCNN_EUNSUPPORTED, "conv_maxpool: geometry not covered by the fused kernel");
  a.src = src;
  a.dst = dst;
  a.workspace = nullptr;
  a.blk = flags;
  if (flags && !lcnn_impl::conv_hwcn32_ok(a, pool_win, pool_stride))
    return fail(LCNN_EUNSUPPORTED, "conv_maxpool: blocked input layout not covered by this route");
  cudaError_t e = lcnn_impl::launch_conv_maxpool_packed(a, d_packed, pool_win, pool_stride,
                                                        S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "conv_maxpool_packed");
  return ok();
}

lcnn_status lcnn_conv_oracle(const float* src, const float* filters, float* dst, uint32_t n,
                             uint32_t c_i, uint32_t h, uint32_t w, int layout, uint32_t c_o,
                             uint32_t f_h, uint32_t f_w, uint32_t stride, uint32_t pad,
                             void* stream) {
  if (!src || !filters || !dst) return fail(LCNN_EINVAL, "conv: null pointer");
  if (!valid_layout(layout)) return fail(LCNN_EINVAL, "conv_oracle: bad layout code");
  lcnn_status st = check_volume(n, c_i, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  st = check_volume(c_o, c_i, f_h, f_w, "FilterBank");
  if (st != LCNN_OK) return st;
  uint32_t ho = 0, wo = 0;
  st = lcnn_conv_output_extents(h, w, f_h, f_w, stride, pad, &ho, &wo);
  if (st != LCNN_OK) return st;
  uint64_t sn, sc, sh, sw;
  switch (layout) {
    case LCNN_NCHW: sw = 1; sh = w; sc = uint64_t{h} * w; sn = uint64_t{c_i} * h * w; break;
    case LCNN_CHWN: sn = 1; sw = n; sh = uint64_t{w} * n; sc = uint64_t{h} * w * n; break;
    case LCNN_NHWC: sc = 1; sw = c_i; sh = uint64_t{w} * c_i; sn = uint64_t{h} * w * c_i; break;
    default: sn = 1; sc = n; sw = uint64_t{c_i} * n; sh = uint64_t{w} * c_i * n; break;
  }
  lcnn_impl::ConvArgs a{src, filters, dst, n, c_i, h, w, c_o, f_h, f_w, stride, pad, ho, wo,
                        layout, LCNN_PREC_FP32, nullptr};
  cudaError_t e = lcnn_impl::launch_conv_oracle(a, sn, sc, sh, sw, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "conv_oracle");
  return ok();
}

lcnn_status lcnn_im2col(const float* src, float* dst, uint32_t n, uint32_t c_i, uint32_t h,
                        uint32_t w, int layout, uint32_t f_h, uint32_t f_w, uint32_t stride,
                        uint32_t pad, void* stream) {
  if (!src || !dst) return fail(LCNN_EINVAL, "im2col: null pointer");
  if (layout != LCNN_NCHW) return fail(LCNN_ELAYOUT, "im2col: input must be NCHW");
  lcnn_status st = check_volume(n, c_i, h, w, "Tensor4D");
  if (st != LCNN_OK) return st;
  uint32_t ho = 0, wo = 0;
  st = lcnn_conv_output_extents(h, w, f_h, f_w, stride, pad, &ho, &wo);
  if (st != LCNN_OK) return st;
  lcnn_impl::ConvArgs a{src, nullptr, dst, n, c_i, h, w, 1, f_h, f_w, stride, pad, ho, wo,
                        layout, LCNN_PREC_FP32, nullptr};
  cudaError_t e = lcnn_impl::launch_im2col(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "im2col");
  return ok();
}

lcnn_status lcnn_gemm(const float* a, const float* b, float* c, uint64_t m, uint64_t n,
                      uint64_t k, int precision, void* d_workspace, size_t workspace_bytes,
                      void* stream) {
  if (!a || !b || !c) return fail(LCNN_EINVAL, "gemm: null pointer");
  if (m == 0 || n == 0 || k == 0) return fail(LCNN_ESHAPE, "gemm: empty operand");
  if (precision < LCNN_PREC_TF32 || precision > LCNN_PREC_FP32)
    return fail(LCNN_EINVAL, "gemm: bad precision");
  cudaError_t e;
  if (precision != LCNN_PREC_FP32 && lcnn_impl::tc_gemm_supported(m, n, k, a, b)) {
    if (workspace_bytes < lcnn_impl::gemm_workspace_bytes(m, n, k, precision))
      return fail(LCNN_EINVAL, "gemm: workspace too small");
    e = lcnn_impl::launch_gemm_tc(a, b, c, m, n, k, precision, d_workspace, S(stream));
  } else {
    e = lcnn_impl::launch_gemm_fp32(a, b, c, m, n, k, S(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "gemm");
  return ok();
}

size_t lcnn_fc_packed_bytes(uint64_t k, uint64_t n, int precision) {
  if (k == 0 || n == 0 || (precision != LCNN_PREC_TF32 && precision != LCNN_PREC_3XTF32)) return 0;
  return lcnn_impl::fc_packed_bytes(k, n, precision);
}

size_t lcnn_fc_workspace_bytes(uint64_t m, uint64_t k, int precision) {
  return lcnn_impl::fc_workspace_bytes(m, k, precision);
}

lcnn_status lcnn_fc_pack_weights(const float* weights, void* d_packed, size_t packed_bytes,
                                 uint64_t k, uint64_t n, int precision, void* stream) {
  if (!weights || !d_packed) return fail(LCNN_EINVAL, "fc: null pointer");
  if (reinterpret_cast<uintptr_t>(d_packed) & 255u)
    return fail(LCNN_EINVAL, "fc: packed weights must be 256-byte aligned");
  if (k == 0 || n == 0) return fail(LCNN_ESHAPE, "gemm: empty operand");
  if (precision != LCNN_PREC_TF32 && precision != LCNN_PREC_3XTF32)
    return fail(LCNN_EINVAL, "fc: packed weights need TF32 or 3xTF32 precision");
  if (packed_bytes < lcnn_impl::fc_packed_bytes(k, n, precision))
    return fail(LCNN_EINVAL, "fc: packed buffer too small");
  cudaError_t e = lcnn_impl::launch_fc_pack(weights, k, n, precision, d_packed, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fc_pack_weights");
  return ok();
}

lcnn_status lcnn_fc_forward_packed(const float* x, int x_layout, const void* d_packed, float* y,
                                   uint64_t m, uint64_t n, uint64_t k, int precision,
                                   void* d_workspace, size_t workspace_bytes, void* stream) {
  return lcnn_fc_forward_packed_ex(x, x_layout, d_packed, y, m, n, k, precision, d_workspace,
                                   workspace_bytes, nullptr, nullptr, 0, stream);
}

lcnn_status lcnn_fc_forward_packed_ex(const float* x, int x_layout, const void* d_packed,
                                      float* y, uint64_t m, uint64_t n, uint64_t k,
                                      int precision, void* d_workspace, size_t workspace_bytes,
                                      void* d_sync, const void* d_next_packed, size_t next_bytes,
                                      void* stream) {
  if (!x || !d_packed || !y) return fail(LCNN_EINVAL, "fc: null pointer");
  if (reinterpret_cast<uintptr_t>(d_sync) & 7u)
    return fail(LCNN_EINVAL, "fc: sync word must be 8-byte aligned");
  if (reinterpret_cast<uintptr_t>(d_packed) & 255u)
    return fail(LCNN_EINVAL, "fc: packed weights must be 256-byte aligned");
  if (m == 0 || n == 0 || k == 0) return fail(LCNN_ESHAPE, "gemm: empty operand");
  if (precision != LCNN_PREC_TF32 && precision != LCNN_PREC_3XTF32)
    return fail(LCNN_EINVAL, "fc: packed weights need TF32 or 3xTF32 precision");
  if (x_layout != LCNN_NCHW && x_layout != LCNN_CHWN)
    return fail(LCNN_ELAYOUT, "fc: input must be NCHW rows or a CHWN tensor");
  const bool a_mn = x_layout == LCNN_CHWN;
  if (!lcnn_impl::fc_tc_supported(m, n, k, a_mn) || (reinterpret_cast<uintptr_t>(x) & 15u))
    return fail(LCNN_EUNSUPPORTED, "fc: shape not supported by the packed tensor-core path");
  if (workspace_bytes < lcnn_impl::fc_workspace_bytes(m, k, precision) ||
      (!d_workspace && workspace_bytes))
    return fail(LCNN_EINVAL, "fc: workspace too small");
  cudaError_t e = lcnn_impl::launch_fc_packed(x, a_mn, d_packed, y, m, n, k, precision,
                                              d_workspace, S(stream),
                                              static_cast<unsigned long long*>(d_sync),
                                              d_next_packed, d_next_packed ? next_bytes : 0);
  if (e != cudaSuccess) return cuda_fail(e, "fc_forward_packed");
  return ok();
}

}  // extern "C"
