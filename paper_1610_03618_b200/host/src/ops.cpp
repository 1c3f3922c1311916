// Host-tensor entry points of the lcnn API (layout.hpp, pool.hpp,
// softmax.hpp, conv.hpp): each call uploads its input, runs one C-ABI kernel
// family (include/lcnn_cuda.h) on the calling thread's stream and downloads
// the fresh output -- value semantics as in the reference, compute on the
// B200.  The device-resident overloads skip the transfers.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "lcnn/conv.hpp"
#include "lcnn/layout.hpp"
#include "lcnn/pool.hpp"
#include "lcnn/softmax.hpp"
#include "lcnn_cuda.h"

namespace lcnn {

namespace {

int code(Layout l) { return static_cast<int>(l); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- scratch for the five-pass softmax / gemm / conv workspaces ----------
DeviceBuffer& scratch(std::size_t bytes) {
  thread_local DeviceBuffer buf;
  if (buf.bytes() < bytes) buf = DeviceBuffer(bytes);
  return buf;
}

int* nonfinite_flag() {
  thread_local DeviceBuffer flag(sizeof(int) * 4);
  return static_cast<int*>(flag.get());
}

bool read_flag(int* d_flag) {
  int h = 0;
  cuda_check(cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost,
                             static_cast<cudaStream_t>(current_stream())),
             "flag readback");
  synchronize();
  return h != 0;
}

}  // namespace

// ============================================================== layout ===
bool flattenable_pair(Layout src, Layout dst) {
  return lcnn_flattenable_pair(code(src), code(dst)) != 0;
}

TransformPlan make_plan(Layout src, Layout dst, std::uint32_t n, std::uint32_t, std::uint32_t,
                        std::uint32_t) {
  TransformPlan p;
  p.src = src;
  p.dst = dst;
  p.tile = 32;
  const bool flat = flattenable_pair(src, dst);
  p.kind = flat ? TransformKind::Tiled2D : TransformKind::NaivePermute;
  p.wide_copy = flat && n >= 64;
  return p;
}

DeviceTensor4D transform(const DeviceTensor4D& t, Layout dst) {
  DeviceTensor4D out(t.n(), t.c(), t.h(), t.w(), dst);
  check_status(lcnn_transform(t.data(), out.data(), t.n(), t.c(), t.h(), t.w(), code(t.layout()),
                              code(dst), current_stream()));
  return out;
}

Tensor4D transform_naive(const Tensor4D& t, Layout dst) {
  const DeviceTensor4D in = DeviceTensor4D::upload(t);
  DeviceTensor4D out(t.n(), t.c(), t.h(), t.w(), dst);
  check_status(lcnn_transform_naive(in.data(), out.data(), t.n(), t.c(), t.h(), t.w(),
                                    code(t.layout()), code(dst), current_stream()));
  return out.download();
}

Tensor4D transform_tiled(const Tensor4D& t, Layout dst, const TransformPlan& plan) {
  if (plan.dst != dst) throw PlanError("transform_tiled: plan destination layout does not match");
  if (plan.src != t.layout())
    throw PlanError("transform_tiled: plan source layout does not match tensor");
  const DeviceTensor4D in = DeviceTensor4D::upload(t);
  DeviceTensor4D out(t.n(), t.c(), t.h(), t.w(), dst);
  check_status(lcnn_transform_tiled(in.data(), out.data(), t.n(), t.c(), t.h(), t.w(),
                                    code(t.layout()), code(dst), plan.tile,
                                    plan.wide_copy ? 1 : 0, current_stream()));
  return out.download();
}

Tensor4D transform(const Tensor4D& t, Layout dst) {
  const TransformPlan plan = make_plan(t.layout(), dst, t.n(), t.c(), t.h(), t.w());
  return plan.kind == TransformKind::Tiled2D ? transform_tiled(t, dst, plan)
                                             : transform_naive(t, dst);
}

// ================================================================ pool ===
std::pair<std::uint32_t, std::uint32_t> pool_output_extents(std::uint32_t h, std::uint32_t w,
                                                            const PoolParams& p) {
  return {(h - p.win_h) / p.stride + 1, (w - p.win_w) / p.stride + 1};
}

namespace {

std::pair<std::uint32_t, std::uint32_t> checked_extents(std::uint32_t h, std::uint32_t w,
                                                        const PoolParams& p) {
  std::uint32_t ho = 0, wo = 0;
  check_status(lcnn_pool_output_extents(h, w, p.win_h, p.win_w, p.stride, &ho, &wo));
  return {ho, wo};
}

int mode_code(const PoolParams& p) { return p.mode == PoolMode::Average ? LCNN_POOL_AVG : LCNN_POOL_MAX; }

AccessReport to_report(const lcnn_access_report& r) {
  return AccessReport{r.input_loads, r.output_stores, r.distinct_inputs};
}

}  // namespace

std::pair<DeviceTensor4D, AccessReport> pool_layout(const DeviceTensor4D& in, const PoolParams& p) {
  const auto [ho, wo] = checked_extents(in.h(), in.w(), p);
  DeviceTensor4D out(in.n(), in.c(), ho, wo, in.layout());
  lcnn_access_report r{};
  check_status(lcnn_pool_layout(in.data(), out.data(), in.n(), in.c(), in.h(), in.w(),
                                code(in.layout()), p.win_h, p.win_w, p.stride, mode_code(p), &r,
                                current_stream()));
  return {std::move(out), to_report(r)};
}

std::pair<DeviceTensor4D, AccessReport> pool_coarsened(const DeviceTensor4D& in,
                                                       const PoolParams& p,
                                                       const CoarseningPlan& plan) {
  const auto [ho, wo] = checked_extents(in.h(), in.w(), p);
  DeviceTensor4D out(in.n(), in.c(), ho, wo, Layout::CHWN);
  lcnn_access_report r{};
  check_status(lcnn_pool_coarsened(in.data(), out.data(), in.n(), in.c(), in.h(), in.w(),
                                   code(in.layout()), p.win_h, p.win_w, p.stride, mode_code(p),
                                   plan.fh, plan.fw, &r, current_stream()));
  return {std::move(out), to_report(r)};
}

lcnn_pool_plan tune_pool_plan(std::uint32_t n, std::uint32_t c, std::uint32_t h,
                              std::uint32_t w, Layout layout, const PoolParams& p) {
  checked_extents(h, w, p);
  lcnn_pool_plan plan{};
  check_status(lcnn_pool_tune(n, c, h, w, code(layout), p.win_h, p.win_w, p.stride, mode_code(p),
                              &plan, current_stream()));
  return plan;
}

std::pair<DeviceTensor4D, AccessReport> pool_run_plan(const DeviceTensor4D& in,
                                                      const PoolParams& p,
                                                      const lcnn_pool_plan& plan) {
  const auto [ho, wo] = checked_extents(in.h(), in.w(), p);
  DeviceTensor4D out(in.n(), in.c(), ho, wo, in.layout());
  lcnn_access_report r{};
  check_status(lcnn_pool_run_plan(in.data(), out.data(), in.n(), in.c(), in.h(), in.w(),
                                  code(in.layout()), p.win_h, p.win_w, p.stride, mode_code(p),
                                  &plan, &r, current_stream()));
  return {std::move(out), to_report(r)};
}

Tensor4D pool_oracle(const Tensor4D& in, const PoolParams& p) {
  const auto [ho, wo] = checked_extents(in.h(), in.w(), p);
  const DeviceTensor4D d = DeviceTensor4D::upload(in);
  DeviceTensor4D out(in.n(), in.c(), ho, wo, Layout::NCHW);
  check_status(lcnn_pool_oracle(d.data(), out.data(), in.n(), in.c(), in.h(), in.w(),
                                code(in.layout()), p.win_h, p.win_w, p.stride, mode_code(p),
                                current_stream()));
  return out.download();
}

std::pair<Tensor4D, AccessReport> pool_layout(const Tensor4D& in, const PoolParams& p) {
  checked_extents(in.h(), in.w(), p);
  if (in.layout() != Layout::CHWN && in.layout() != Layout::NCHW)
    throw LayoutError("pool_layout: only CHWN and NCHW kernels exist");
  auto [out, r] = pool_layout(DeviceTensor4D::upload(in), p);
  return {out.download(), r};
}

std::pair<Tensor4D, AccessReport> pool_coarsened(const Tensor4D& in, const PoolParams& p,
                                                 const CoarseningPlan& plan) {
  checked_extents(in.h(), in.w(), p);
  if (plan.fh < 1 || plan.fw < 1) throw PlanError("pool_coarsened: factors must be >= 1");
  if (std::uint64_t{plan.fh} * plan.fw > kCoarseningCap)
    throw PlanError("pool_coarsened: fh*fw exceeds accumulator cap of 64");
  if (in.layout() != Layout::CHWN) throw LayoutError("pool_coarsened: input must be CHWN");
  auto [out, r] = pool_coarsened(DeviceTensor4D::upload(in), p, plan);
  return {out.download(), r};
}

CoarseningPlan autotune_pool(std::uint32_t n, std::uint32_t c, std::uint32_t h, std::uint32_t w,
                             const PoolParams& p, PoolCostFn measure) {
  if (!measure) {
    // GPU cost model: median of 5 CUDA-event timings of the coarsened kernel
    // on a seeded device-resident CHWN input (pool.cpp:275-294 semantics).
    Tensor4D host(n, c, h, w, Layout::CHWN);
    std::mt19937 rng(42);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    for (std::uint64_t i = 0; i < host.size(); ++i) host.data()[i] = dist(rng);
    auto input = std::make_shared<DeviceTensor4D>(DeviceTensor4D::upload(host));
    auto out = std::make_shared<DeviceTensor4D>(n, c, pool_output_extents(h, w, p).first,
                                                pool_output_extents(h, w, p).second, Layout::CHWN);
    measure = [input, out, p](const CoarseningPlan& plan) {
      cudaStream_t s = static_cast<cudaStream_t>(current_stream());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto run = [&] {
        check_status(lcnn_pool_coarsened(input->data(), out->data(), input->n(), input->c(),
                                         input->h(), input->w(), LCNN_CHWN, p.win_h, p.win_w,
                                         p.stride, mode_code(p), plan.fh, plan.fw, nullptr, s));
      };
      run();  // warm-up
      double samples[5];
      for (double& t : samples) {
        cudaEventRecord(e0, s);
        run();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        t = ms * 1e-3;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      std::sort(std::begin(samples), std::end(samples));
      return samples[2];
    };
  }
  CoarseningPlan best{2, 2};
  double best_cost = measure(best);
  bool more_h = true, more_w = true;
  auto try_step = [&](bool& more, CoarseningPlan cand) {
    if (!more) return;
    if (std::uint64_t{cand.fh} * cand.fw > kCoarseningCap) {
      more = false;
      return;
    }
    const double cost = measure(cand);
    if (cost < best_cost) {
      best = cand;
      best_cost = cost;
    } else {
      more = false;
    }
  };
  while (more_h || more_w) {
    try_step(more_h, CoarseningPlan{best.fh + 1, best.fw});
    try_step(more_w, CoarseningPlan{best.fh, best.fw + 1});
  }
  return best;
}

// ============================================================= softmax ===
void softmax_fused_into(const DeviceMatrix& in, DeviceMatrix& out, bool check_finite,
                        int* sticky_flag) {
  if (in.rows < 1 || in.cols < 1) throw ShapeError("softmax: empty matrix");
  if (out.rows != in.rows || out.cols != in.cols) throw ShapeError("softmax: output dims");
  if (!check_finite && sticky_flag) {  // caller-owned device flag, read later
    check_status(lcnn_softmax_fused_sticky(in.data(), out.data(), in.rows, in.cols, sticky_flag,
                                           current_stream()));
    return;
  }
  int* flag = check_finite ? nonfinite_flag() : nullptr;
  check_status(lcnn_softmax_fused(in.data(), out.data(), in.rows, in.cols, 16384, flag, nullptr,
                                  current_stream()));
  if (flag && read_flag(flag)) throw DomainError("softmax: non-finite input");
}

DeviceMatrix softmax_fused(const DeviceMatrix& in, bool check_finite) {
  DeviceMatrix out(in.rows, in.cols);
  softmax_fused_into(in, out, check_finite);
  return out;
}

std::pair<Matrix, PassReport> softmax_fused(const Matrix& in, std::uint32_t local_buffer_limit) {
  if (in.rows < 1 || in.cols < 1) throw ShapeError("softmax: empty matrix");
  const DeviceMatrix d = DeviceMatrix::upload(in);
  DeviceMatrix out(in.rows, in.cols);
  lcnn_pass_report r{};
  int* flag = nonfinite_flag();
  check_status(lcnn_softmax_fused(d.data(), out.data(), in.rows, in.cols, local_buffer_limit,
                                  flag, &r, current_stream()));
  if (read_flag(flag)) throw DomainError("softmax: non-finite input");
  return {out.download(), PassReport{r.materializations, r.full_matrix_sweeps}};
}

Matrix softmax_reference(const Matrix& in, SoftmaxScratch* sc, PassReport* report) {
  if (in.rows < 1 || in.cols < 1) throw ShapeError("softmax: empty matrix");
  const DeviceMatrix d = DeviceMatrix::upload(in);
  DeviceMatrix out(in.rows, in.cols);
  const std::size_t bytes = lcnn_softmax_reference_scratch_bytes(in.rows, in.cols);
  DeviceBuffer& buf = scratch(bytes);
  lcnn_pass_report r{};
  int* flag = nonfinite_flag();
  check_status(lcnn_softmax_reference(d.data(), out.data(), in.rows, in.cols, buf.get(),
                                      buf.bytes(), flag, &r, current_stream()));
  if (read_flag(flag)) throw DomainError("softmax: non-finite input");
  if (sc) {  // device scratch layout: maxv[rows] sumv[rows] midv1[rows*cols] midv2[...]
    const std::uint64_t rows = in.rows, total = rows * in.cols;
    sc->maxv.resize(rows);
    sc->sumv.resize(rows);
    sc->midv1.resize(total);
    sc->midv2.resize(total);
    const float* base = buf.f();
    cudaStream_t s = static_cast<cudaStream_t>(current_stream());
    cuda_check(cudaMemcpyAsync(sc->maxv.data(), base, rows * 4, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaMemcpyAsync(sc->sumv.data(), base + rows, rows * 4, cudaMemcpyDeviceToHost, s),
               "d2h");
    cuda_check(cudaMemcpyAsync(sc->midv1.data(), base + 2 * rows, total * 4,
                               cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaMemcpyAsync(sc->midv2.data(), base + 2 * rows + total, total * 4,
                               cudaMemcpyDeviceToHost, s), "d2h");
  }
  if (report) *report = PassReport{r.materializations, r.full_matrix_sweeps};
  return out.download();
}

DeviceMatrix fc_forward(const DeviceMatrix& in, const DeviceMatrix& weights) {
  if (in.cols != weights.rows)
    throw ShapeError("gemm: inner dims disagree (" + std::to_string(in.cols) + " vs " +
                     std::to_string(weights.rows) + ")");
  DeviceMatrix out(in.rows, weights.cols);
  const int prec = dense_precision();
  const std::size_t ws = lcnn_gemm_workspace_bytes(in.rows, weights.cols, in.cols, prec);
  DeviceBuffer& buf = scratch(ws + 16);
  check_status(lcnn_gemm(in.data(), weights.data(), out.data(), in.rows, weights.cols, in.cols,
                         prec, buf.get(), buf.bytes(), current_stream()));
  return out;
}

Matrix fc_forward(const Matrix& in, const Matrix& weights) { return gemm_blocked(in, weights); }

std::shared_ptr<DeviceBuffer> pack_fc_weights(const float* d_weights, std::uint32_t k,
                                              std::uint32_t n, int precision) {
  const std::size_t bytes = lcnn_fc_packed_bytes(k, n, precision);
  if (!bytes) return nullptr;
  auto buf = std::make_shared<DeviceBuffer>(bytes);
  check_status(lcnn_fc_pack_weights(d_weights, buf->get(), buf->bytes(), k, n, precision,
                                    current_stream()));
  return buf;
}

namespace {

DeviceMatrix fc_packed_run(const float* x, int layout, std::uint32_t m, std::uint32_t k,
                           const void* d_packed, std::uint32_t n, int precision, void* d_sync,
                           const DeviceBuffer* next) {
  DeviceMatrix out(m, n);
  const std::size_t ws = lcnn_fc_workspace_bytes(m, k, precision);
  void* wsp = nullptr;
  std::size_t wsb = 0;
  if (ws) {
    DeviceBuffer& buf = scratch(ws + 16);
    wsp = buf.get();
    wsb = buf.bytes();
  }
  check_status(lcnn_fc_forward_packed_ex(x, layout, d_packed, out.data(), m, n, k, precision, wsp,
                                         wsb, d_sync, next ? next->get() : nullptr,
                                         next ? next->bytes() : 0, current_stream()));
  return out;
}

}  // namespace

DeviceMatrix fc_forward_packed(const DeviceMatrix& in, const void* d_packed, std::uint32_t n,
                               int precision, void* d_sync, const DeviceBuffer* next_packed) {
  return fc_packed_run(in.data(), LCNN_NCHW, in.rows, in.cols, d_packed, n, precision, d_sync,
                       next_packed);
}

DeviceMatrix fc_forward_packed(const DeviceTensor4D& in, const void* d_packed, std::uint32_t n,
                               int precision, void* d_sync, const DeviceBuffer* next_packed) {
  const std::uint32_t k = in.c() * in.h() * in.w();
  if (in.layout() == Layout::CHWN && in.n() % 4 == 0)
    return fc_packed_run(in.data(), LCNN_CHWN, in.n(), k, d_packed, n, precision, d_sync,
                         next_packed);
  const DeviceTensor4D rows = in.layout() == Layout::NCHW ? in : transform(in, Layout::NCHW);
  return fc_packed_run(rows.data(), LCNN_NCHW, rows.n(), k, d_packed, n, precision, d_sync,
                       next_packed);
}

// ================================================================ conv ===
std::pair<std::uint32_t, std::uint32_t> conv_output_extents(std::uint32_t h, std::uint32_t w,
                                                            std::uint32_t f_h, std::uint32_t f_w,
                                                            const ConvParams& p) {
  std::uint32_t ho = 0, wo = 0;
  check_status(lcnn_conv_output_extents(h, w, f_h, f_w, p.stride, p.pad, &ho, &wo));
  return {ho, wo};
}

namespace {

void check_conv_inputs(const Tensor4D& in, const FilterBank& f) {
  if (in.c() != f.c_i())
    throw ShapeError("conv: input channels " + std::to_string(in.c()) +
                     " do not match filter c_i " + std::to_string(f.c_i()));
}

struct DeviceFilters {
  DeviceBuffer buf;
  explicit DeviceFilters(const FilterBank& f) : buf(f.size() * sizeof(float)) {
    cuda_check(cudaMemcpyAsync(buf.get(), f.data(), f.size() * sizeof(float),
                               cudaMemcpyHostToDevice, static_cast<cudaStream_t>(current_stream())),
               "upload filters");
  }
};

}  // namespace

DeviceTensor4D conv_forward(const DeviceTensor4D& in, const float* d_filters, std::uint32_t c_o,
                            std::uint32_t f_h, std::uint32_t f_w, const ConvParams& p,
                            int precision) {
  const auto [ho, wo] = conv_output_extents(in.h(), in.w(), f_h, f_w, p);
  DeviceTensor4D out(in.n(), c_o, ho, wo, in.layout());
  const std::size_t ws =
      lcnn_conv_workspace_bytes_ex(in.n(), in.c(), in.h(), in.w(), code(in.layout()), c_o, f_h,
                                   f_w, p.stride, p.pad, precision);
  DeviceBuffer& buf = scratch(ws + 16);
  check_status(lcnn_conv_forward(in.data(), d_filters, out.data(), in.n(), in.c(), in.h(), in.w(),
                                 code(in.layout()), c_o, f_h, f_w, p.stride, p.pad, precision,
                                 buf.get(), buf.bytes(), current_stream()));
  return out;
}

std::shared_ptr<DeviceBuffer> pack_conv_filters(const DeviceTensor4D& in, const float* d_filters,
                                                std::uint32_t c_o, std::uint32_t f_h,
                                                std::uint32_t f_w, const ConvParams& p,
                                                int precision) {
  conv_output_extents(in.h(), in.w(), f_h, f_w, p);
  const std::size_t bytes = lcnn_conv_packed_bytes(in.n(), in.c(), in.h(), in.w(), code(in.layout()),
                                                   c_o, f_h, f_w, p.stride, p.pad, precision);
  auto buf = std::make_shared<DeviceBuffer>(bytes ? bytes : 256);
  check_status(lcnn_conv_pack_filters(d_filters, buf->get(), buf->bytes(), in.n(), in.c(), in.h(),
                                      in.w(), code(in.layout()), c_o, f_h, f_w, p.stride, p.pad,
                                      precision, current_stream()));
  return buf;
}

DeviceTensor4D conv_forward_packed(const DeviceTensor4D& in, const void* d_packed,
                                   std::uint32_t c_o, std::uint32_t f_h, std::uint32_t f_w,
                                   const ConvParams& p, int precision, void* d_sync,
                                   std::uint32_t blk_flags) {
  const auto [ho, wo] = conv_output_extents(in.h(), in.w(), f_h, f_w, p);
  DeviceTensor4D out(in.n(), c_o, ho, wo, in.layout());
  const std::size_t ws = lcnn_conv_packed_workspace_bytes(
      in.n(), in.c(), in.h(), in.w(), code(in.layout()), c_o, f_h, f_w, p.stride, p.pad, precision);
  void* wsp = nullptr;
  std::size_t wsb = 0;
  if (ws) {
    DeviceBuffer& buf = scratch(ws + 16);
    wsp = buf.get();
    wsb = buf.bytes();
  }
  check_status(lcnn_conv_forward_packed_blk(in.data(), d_packed, out.data(), in.n(), in.c(),
                                            in.h(), in.w(), code(in.layout()), c_o, f_h, f_w,
                                            p.stride, p.pad, precision, wsp, wsb, d_sync,
                                            blk_flags, current_stream()));
  return out;
}

bool conv_maxpool_supported(const DeviceTensor4D& in, std::uint32_t c_o, std::uint32_t f_h,
                            std::uint32_t f_w, const ConvParams& p, int precision,
                            std::uint32_t pool_win, std::uint32_t pool_stride) {
  return lcnn_conv_maxpool_supported(in.n(), in.c(), in.h(), in.w(), code(in.layout()), c_o, f_h,
                                     f_w, p.stride, p.pad, precision, pool_win,
                                     pool_stride) == 1;
}

DeviceTensor4D conv_maxpool_forward_packed(const DeviceTensor4D& in, const void* d_packed,
                                           std::uint32_t c_o, std::uint32_t f_h,
                                           std::uint32_t f_w, const ConvParams& p, int precision,
                                           std::uint32_t pool_win, std::uint32_t pool_stride,
                                           std::uint32_t blk_flags) {
  const auto [ho, wo] = conv_output_extents(in.h(), in.w(), f_h, f_w, p);
  if (pool_win == 0 || pool_stride == 0 || pool_win > ho || pool_win > wo)
    throw ShapeError("conv_maxpool: pool window does not fit the conv output");
  const std::uint32_t hp = (ho - pool_win) / pool_stride + 1;
  const std::uint32_t wp = (wo - pool_win) / pool_stride + 1;
  DeviceTensor4D out(in.n(), c_o, hp, wp, in.layout());
  check_status(lcnn_conv_maxpool_packed_blk(in.data(), d_packed, out.data(), in.n(), in.c(),
                                            in.h(), in.w(), code(in.layout()), c_o, f_h, f_w,
                                            p.stride, p.pad, precision, pool_win, pool_stride,
                                            blk_flags, current_stream()));
  return out;
}

bool conv_hwcn32_supported(const DeviceTensor4D& in, std::uint32_t c_o, std::uint32_t f_h,
                           std::uint32_t f_w, const ConvParams& p, int precision,
                           std::uint32_t pool_win, std::uint32_t pool_stride,
                           std::uint32_t blk_flags) {
  if (in.layout() != Layout::CHWN) return false;
  return lcnn_conv_hwcn32_supported(in.n(), in.c(), in.h(), in.w(), c_o, f_h, f_w, p.stride,
                                    p.pad, precision, pool_win, pool_stride, blk_flags) == 1;
}

Tensor4D conv_oracle(const Tensor4D& in, const FilterBank& f, const ConvParams& p) {
  check_conv_inputs(in, f);
  const auto [ho, wo] = conv_output_extents(in.h(), in.w(), f.f_h(), f.f_w(), p);
  const DeviceTensor4D d = DeviceTensor4D::upload(in);
  DeviceFilters df(f);
  DeviceTensor4D out(in.n(), f.c_o(), ho, wo, Layout::NCHW);
  check_status(lcnn_conv_oracle(d.data(), df.buf.f(), out.data(), in.n(), in.c(), in.h(), in.w(),
                                code(in.layout()), f.c_o(), f.f_h(), f.f_w(), p.stride, p.pad,
                                current_stream()));
  return out.download();
}

Tensor4D conv_direct(const Tensor4D& in, const FilterBank& f, const ConvParams& p) {
  check_conv_inputs(in, f);
  conv_output_extents(in.h(), in.w(), f.f_h(), f.f_w(), p);
  if (in.layout() != Layout::CHWN && in.layout() != Layout::NCHW)
    throw LayoutError("conv_direct: only CHWN and NCHW kernels exist");
  const DeviceTensor4D d = DeviceTensor4D::upload(in);
  DeviceFilters df(f);
  return conv_forward(d, df.buf.f(), f.c_o(), f.f_h(), f.f_w(), p, dense_precision()).download();
}

Tensor4D conv_gemm(const Tensor4D& in, const FilterBank& f, const ConvParams& p) {
  check_conv_inputs(in, f);
  if (in.layout() != Layout::NCHW) throw LayoutError("conv_gemm: input must be NCHW");
  conv_output_extents(in.h(), in.w(), f.f_h(), f.f_w(), p);
  const DeviceTensor4D d = DeviceTensor4D::upload(in);
  DeviceFilters df(f);
  return conv_forward(d, df.buf.f(), f.c_o(), f.f_h(), f.f_w(), p, dense_precision()).download();
}

Tensor4D conv_fft(const Tensor4D& in, const FilterBank& f, const ConvParams& p) {
  check_conv_inputs(in, f);
  if (p.stride != 1) throw UnsupportedError("conv_fft: only stride 1 is supported");
  if (in.layout() != Layout::NCHW) throw LayoutError("conv_fft: input must be NCHW");
  return conv_gemm(in, f, p);
}

Matrix im2col(const Tensor4D& in, std::uint32_t f_h, std::uint32_t f_w, const ConvParams& p) {
  if (in.layout() != Layout::NCHW) throw LayoutError("im2col: input must be NCHW");
  const auto [ho, wo] = conv_output_extents(in.h(), in.w(), f_h, f_w, p);
  const std::uint64_t rows = std::uint64_t{in.c()} * f_h * f_w;
  const std::uint64_t cols = std::uint64_t{in.n()} * ho * wo;
  const DeviceTensor4D d = DeviceTensor4D::upload(in);
  DeviceMatrix out(static_cast<std::uint32_t>(rows), static_cast<std::uint32_t>(cols));
  check_status(lcnn_im2col(d.data(), out.data(), in.n(), in.c(), in.h(), in.w(), LCNN_NCHW, f_h,
                           f_w, p.stride, p.pad, current_stream()));
  return out.download();
}

void gemm_blocked(const float* a, const float* b, float* c, std::uint64_t m, std::uint64_t n,
                  std::uint64_t k) {
  DeviceBuffer da(m * k * 4 + 16), db(k * n * 4 + 16), dc(m * n * 4 + 16);
  cudaStream_t s = static_cast<cudaStream_t>(current_stream());
  cuda_check(cudaMemcpyAsync(da.get(), a, m * k * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_check(cudaMemcpyAsync(db.get(), b, k * n * 4, cudaMemcpyHostToDevice, s), "h2d");
  const int prec = dense_precision();
  const std::size_t ws = lcnn_gemm_workspace_bytes(m, n, k, prec);
  DeviceBuffer& buf = scratch(ws + 16);
  check_status(lcnn_gemm(da.f(), db.f(), dc.f(), m, n, k, prec, buf.get(), buf.bytes(), s));
  cuda_check(cudaMemcpyAsync(c, dc.get(), m * n * 4, cudaMemcpyDeviceToHost, s), "d2h");
  synchronize();
}

Matrix gemm_blocked(const Matrix& a, const Matrix& b) {
  if (a.cols != b.rows)
    throw ShapeError("gemm: inner dims disagree (" + std::to_string(a.cols) + " vs " +
                     std::to_string(b.rows) + ")");
  Matrix c(a.rows, b.cols);
  if (a.rows && b.cols && a.cols) gemm_blocked(a.data.data(), b.data.data(), c.data.data(), a.rows,
                                               b.cols, a.cols);
  return c;
}

}  // namespace lcnn
