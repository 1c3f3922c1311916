// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library, compiled from
// the sources where they lie (/root/reference/proj/src, see oracle/Makefile)
// with -Dlcnn=lcnn_ref so the reference namespace cannot collide with
// anything else.  Output: oracle/_ref/liblcnn_ref.so (git-ignored; travels to
// the GPU box with the snapshot).  Used to
//   * pin the C restatement (oracle/lcnn_oracle.c) to the real reference,
//   * generate the golden fixtures in tests/golden/ (tests/golden/make_golden.py),
//   * time the reference CPU path for bench.py (cpu_baseline and
//     --impl reference), optionally one std::thread per N-shard.
// Status codes are the lcnn_status values of include/lcnn_cuda.h.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "lcnn/conv.hpp"
#include "lcnn/fixtures.hpp"
#include "lcnn/layout.hpp"
#include "lcnn/net.hpp"
#include "lcnn/pool.hpp"
#include "lcnn/select.hpp"
#include "lcnn/softmax.hpp"
#include "lcnn/tensor.hpp"

namespace R = lcnn_ref;

namespace {

thread_local std::string g_err;

int map_current_exception() {
  try {
    throw;
  } catch (const R::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const R::IndexError& e) {
    g_err = e.what();
    return 2;
  } catch (const R::LayoutError& e) {
    g_err = e.what();
    return 3;
  } catch (const R::PlanError& e) {
    g_err = e.what();
    return 4;
  } catch (const R::FormatError& e) {
    g_err = e.what();
    return 5;
  } catch (const R::DomainError& e) {
    g_err = e.what();
    return 6;
  } catch (const R::UnsupportedError& e) {
    g_err = e.what();
    return 7;
  } catch (const R::ValidationError& e) {
    g_err = e.what();
    return 8;
  } catch (const R::CalibrationError& e) {
    g_err = e.what();
    return 9;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 11;
  } catch (...) {
    g_err = "unknown exception";
    return 11;
  }
}

R::Tensor4D make_tensor(const float* p, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                        int layout) {
  const uint64_t size = uint64_t{n} * c * h * w;
  return R::Tensor4D(n, c, h, w, static_cast<R::Layout>(layout),
                     std::vector<float>(p, p + size));
}

void copy_out(const R::Tensor4D& t, float* dst) {
  std::memcpy(dst, t.data(), t.size() * sizeof(float));
}

R::Matrix make_matrix(const float* p, uint32_t rows, uint32_t cols) {
  R::Matrix m(rows, cols);
  std::memcpy(m.data.data(), p, m.data.size() * sizeof(float));
  return m;
}

void fill_report(const R::AccessReport& r, uint64_t* out) {
  if (!out) return;
  out[0] = r.input_loads;
  out[1] = r.output_stores;
  out[2] = r.distinct_inputs;
}

}  // namespace

#define GUARD(...)                      \
  try {                                \
    __VA_ARGS__;                       \
    g_err.clear();                     \
    return 0;                          \
  } catch (...) {                      \
    return map_current_exception();    \
  }

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_transform(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                  int sl, int dl) {
  GUARD(copy_out(R::transform(make_tensor(src, n, c, h, w, sl), static_cast<R::Layout>(dl)), dst))
}

int ref_transform_naive(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                        uint32_t w, int sl, int dl) {
  GUARD(copy_out(R::transform_naive(make_tensor(src, n, c, h, w, sl), static_cast<R::Layout>(dl)),
                 dst))
}

int ref_transform_tiled(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                        uint32_t w, int sl, int dl, uint32_t tile, int wide) {
  GUARD({
    R::TransformPlan plan = R::make_plan(static_cast<R::Layout>(sl), static_cast<R::Layout>(dl), n,
                                         c, h, w);
    plan.tile = tile;
    plan.wide_copy = wide != 0;
    plan.kind = R::TransformKind::Tiled2D;
    copy_out(R::transform_tiled(make_tensor(src, n, c, h, w, sl), static_cast<R::Layout>(dl), plan),
             dst);
  })
}

int ref_make_plan(int sl, int dl, uint32_t n, uint32_t c, uint32_t h, uint32_t w, int* kind,
                  uint32_t* tile, int* wide) {
  GUARD({
    const R::TransformPlan p =
        R::make_plan(static_cast<R::Layout>(sl), static_cast<R::Layout>(dl), n, c, h, w);
    *kind = static_cast<int>(p.kind);
    *tile = p.tile;
    *wide = p.wide_copy ? 1 : 0;
  })
}

int ref_pool_oracle(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg) {
  GUARD(copy_out(R::pool_oracle(make_tensor(src, n, c, h, w, layout),
                                R::PoolParams{wh, ww, s, avg ? R::PoolMode::Average : R::PoolMode::Max}),
                 dst))
}

int ref_pool_layout(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg, uint64_t* report) {
  GUARD({
    auto r = R::pool_layout(make_tensor(src, n, c, h, w, layout),
                            R::PoolParams{wh, ww, s, avg ? R::PoolMode::Average : R::PoolMode::Max});
    copy_out(r.first, dst);
    fill_report(r.second, report);
  })
}

int ref_pool_coarsened(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                       uint32_t w, int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg,
                       uint32_t fh, uint32_t fw, uint64_t* report) {
  GUARD({
    auto r = R::pool_coarsened(make_tensor(src, n, c, h, w, layout),
                               R::PoolParams{wh, ww, s, avg ? R::PoolMode::Average : R::PoolMode::Max},
                               R::CoarseningPlan{fh, fw});
    copy_out(r.first, dst);
    fill_report(r.second, report);
  })
}

typedef double (*ref_cost_fn)(uint32_t fh, uint32_t fw, void* ctx);
int ref_autotune_pool(uint32_t n, uint32_t c, uint32_t h, uint32_t w, uint32_t wh, uint32_t ww,
                      uint32_t s, int avg, ref_cost_fn cost, void* ctx, uint32_t* fh,
                      uint32_t* fw) {
  GUARD({
    R::PoolCostFn fn;
    if (cost) fn = [cost, ctx](const R::CoarseningPlan& p) { return cost(p.fh, p.fw, ctx); };
    const R::CoarseningPlan p = R::autotune_pool(
        n, c, h, w, R::PoolParams{wh, ww, s, avg ? R::PoolMode::Average : R::PoolMode::Max}, fn);
    *fh = p.fh;
    *fw = p.fw;
  })
}

int ref_softmax_reference(const float* in, float* out, uint32_t rows, uint32_t cols,
                          uint32_t* report) {
  GUARD({
    R::PassReport rep;
    const R::Matrix o = R::softmax_reference(make_matrix(in, rows, cols), nullptr, &rep);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    if (report) {
      report[0] = rep.materializations;
      report[1] = rep.full_matrix_sweeps;
    }
  })
}

int ref_softmax_fused(const float* in, float* out, uint32_t rows, uint32_t cols, uint32_t limit,
                      uint32_t* report) {
  GUARD({
    auto r = R::softmax_fused(make_matrix(in, rows, cols), limit);
    std::memcpy(out, r.first.data.data(), r.first.data.size() * sizeof(float));
    if (report) {
      report[0] = r.second.materializations;
      report[1] = r.second.full_matrix_sweeps;
    }
  })
}

int ref_conv_oracle(const float* in, const float* filt, float* out, uint32_t n, uint32_t ci,
                    uint32_t h, uint32_t w, int layout, uint32_t co, uint32_t fh, uint32_t fw,
                    uint32_t stride, uint32_t pad) {
  GUARD({
    R::FilterBank f(co, ci, fh, fw,
                    std::vector<float>(filt, filt + uint64_t{co} * ci * fh * fw));
    copy_out(R::conv_oracle(make_tensor(in, n, ci, h, w, layout), f, R::ConvParams{stride, pad}),
             out);
  })
}

int ref_conv_direct(const float* in, const float* filt, float* out, uint32_t n, uint32_t ci,
                    uint32_t h, uint32_t w, int layout, uint32_t co, uint32_t fh, uint32_t fw,
                    uint32_t stride, uint32_t pad) {
  GUARD({
    R::FilterBank f(co, ci, fh, fw,
                    std::vector<float>(filt, filt + uint64_t{co} * ci * fh * fw));
    copy_out(R::conv_direct(make_tensor(in, n, ci, h, w, layout), f, R::ConvParams{stride, pad}),
             out);
  })
}

int ref_conv_gemm(const float* in, const float* filt, float* out, uint32_t n, uint32_t ci,
                  uint32_t h, uint32_t w, uint32_t co, uint32_t fh, uint32_t fw, uint32_t stride,
                  uint32_t pad) {
  GUARD({
    R::FilterBank f(co, ci, fh, fw,
                    std::vector<float>(filt, filt + uint64_t{co} * ci * fh * fw));
    copy_out(R::conv_gemm(make_tensor(in, n, ci, h, w, 0), f, R::ConvParams{stride, pad}), out);
  })
}

int ref_gemm_blocked(const float* a, const float* b, float* c, uint64_t m, uint64_t n, uint64_t k) {
  GUARD(R::gemm_blocked(a, b, c, m, n, k))
}

int ref_choose_layout(int kind, uint32_t n, uint32_t c, uint32_t c_t, uint32_t n_t) {
  return static_cast<int>(
      R::choose_layout(static_cast<R::LayerKind>(kind), n, c, R::HeuristicThresholds{c_t, n_t}));
}

typedef double (*ref_bench_fn)(int layout, uint32_t n, uint32_t c, void* ctx);
int ref_calibrate(ref_bench_fn bench, void* ctx, uint32_t* c_t, uint32_t* n_t) {
  GUARD({
    const R::HeuristicThresholds th = R::calibrate(
        [bench, ctx](R::Layout l, uint32_t n, uint32_t c) {
          const double v = bench(static_cast<int>(l), n, c, ctx);
          if (v < 0) throw std::runtime_error("bench exploded");
          return v;
        });
    *c_t = th.c_t;
    *n_t = th.n_t;
  })
}

// parse_network + annotate_layouts (preset c_t/n_t; c_t == 0 keeps explicit
// fields only) + plan_transforms.  layouts_out: one code per layer (-1 for
// layers without a layout).  Returns the number of transform steps via
// *steps and writes (position, src, dst) triples.
int ref_plan_network(const char* json, uint32_t c_t, uint32_t n_t, int* layouts_out,
                     int max_layers, int* steps, int* pos, int* src, int* dst, int max_steps) {
  GUARD({
    R::NetworkSpec spec = R::parse_network(json);
    if (c_t) spec = R::annotate_layouts(spec, R::HeuristicThresholds{c_t, n_t});
    for (int i = 0; i < max_layers && i < static_cast<int>(spec.layers.size()); ++i)
      layouts_out[i] = spec.layers[i].layout_field ? static_cast<int>(*spec.layers[i].layout_field) : -1;
    const auto plan = R::plan_transforms(spec);
    *steps = static_cast<int>(plan.size());
    for (int i = 0; i < max_steps && i < static_cast<int>(plan.size()); ++i) {
      pos[i] = static_cast<int>(plan[i].position);
      src[i] = static_cast<int>(plan[i].src);
      dst[i] = static_cast<int>(plan[i].dst);
    }
  })
}

// --- timing of the reference CPU path (bench.py cpu_baseline / --impl reference)
// op: 0 pool_layout, 1 pool_coarsened(fh,fw), 2 softmax_fused, 3 softmax_reference,
//     4 transform (make_plan dispatch), 5 transform_naive
// A session splits the batch into `threads` disjoint N-shards (n/threads
// images, the last takes the remainder) and builds each shard's seeded input
// once.  ref_session_run starts one std::thread per shard, each running the
// unmodified reference call on its shard, joins them and returns that wall
// interval in seconds.  For the softmax ops n = rows and c = cols.
struct RefSession {
  int op;
  int dst_layout;
  R::PoolParams pp;
  R::CoarseningPlan plan;
  std::vector<R::Tensor4D> tins;
  std::vector<R::Matrix> mins;
  int threads;
};

void* ref_session_create(int op, uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout,
                         int dst_layout, uint32_t wh, uint32_t ww, uint32_t s, int avg,
                         uint32_t fh, uint32_t fw, int threads) {
  try {
    if (threads < 1) threads = 1;
    if (static_cast<uint32_t>(threads) > n) threads = static_cast<int>(n);
    auto* S = new RefSession{op, dst_layout,
                             R::PoolParams{wh, ww, s, avg ? R::PoolMode::Average : R::PoolMode::Max},
                             R::CoarseningPlan{fh, fw}, {}, {}, threads};
    // shard inputs are allocated here and filled in parallel (one thread per
    // shard, seed 42 + t) so a multi-GB session (VGG pool1 at N=256) is ready
    // in about a second
    const uint32_t base = n / threads;
    for (int t = 0; t < threads; ++t) {
      const uint32_t nn = t == threads - 1 ? n - base * (threads - 1) : base;
      if (op == 2 || op == 3)
        S->mins.emplace_back(nn, c);
      else
        S->tins.emplace_back(nn, c, h, w, static_cast<R::Layout>(layout));
    }
    auto fill = [&](int t) {
      std::mt19937 rng(42 + t);
      std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
      if (op == 2 || op == 3) {
        for (auto& v : S->mins[t].data) v = dist(rng);
      } else {
        R::Tensor4D& in = S->tins[t];
        for (uint64_t i = 0; i < in.size(); ++i) in.data()[i] = dist(rng);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(fill, t);
    fill(0);
    for (auto& th : pool) th.join();
    return S;
  } catch (...) {
    map_current_exception();
    return nullptr;
  }
}

double ref_session_run(void* handle) {
  auto* S = static_cast<RefSession*>(handle);
  try {
    auto call = [S](int t) {
      switch (S->op) {
        case 0: (void)R::pool_layout(S->tins[t], S->pp); break;
        case 1: (void)R::pool_coarsened(S->tins[t], S->pp, S->plan); break;
        case 2: (void)R::softmax_fused(S->mins[t]); break;
        case 3: (void)R::softmax_reference(S->mins[t]); break;
        case 4: (void)R::transform(S->tins[t], static_cast<R::Layout>(S->dst_layout)); break;
        default: (void)R::transform_naive(S->tins[t], static_cast<R::Layout>(S->dst_layout)); break;
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < S->threads; ++t) pool.emplace_back(call, t);
    call(0);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } catch (...) {
    map_current_exception();
    return -1.0;
  }
}

void ref_session_destroy(void* handle) { delete static_cast<RefSession*>(handle); }

// Whole-network reference forward: `threads` std::threads, each parsing the
// config (batch = its shard), annotating with (c_t, n_t) and calling the
// unmodified run_network on a seeded input of the first 4D layer's layout.
// Returns the wall seconds of the slowest thread's run_network (inputs and
// weights built before timing).
double ref_time_network(const char* json, uint32_t c_t, uint32_t n_t, int threads) {
  try {
    if (threads < 1) threads = 1;
    std::vector<double> secs(threads, 0.0);
    std::vector<std::string> errs(threads);
    auto work = [&](int t) {
      try {
        R::NetworkSpec spec = R::annotate_layouts(R::parse_network(json),
                                                  R::HeuristicThresholds{c_t, n_t});
        R::Layout first = R::Layout::NCHW;
        for (const auto& l : spec.layers)
          if ((l.kind == R::LayerKind::Convolution || l.kind == R::LayerKind::Pooling) &&
              l.layout_field) {
            first = *l.layout_field;
            break;
          }
        R::Tensor4D in(spec.n, spec.c, spec.h, spec.w, first);
        std::mt19937 rng(42 + t);
        std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
        for (uint64_t i = 0; i < in.size(); ++i) in.data()[i] = dist(rng);
        const auto t0 = std::chrono::steady_clock::now();
        (void)R::run_network(spec, in);
        secs[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      } catch (const std::exception& e) {
        errs[t] = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    return *std::max_element(secs.begin(), secs.end());
  } catch (...) {
    map_current_exception();
    return -1.0;
  }
}

// The unmodified run_network (net.cpp:266-398) on a caller-supplied input in
// `in_layout` (flat order of that layout), network annotated with (c_t, n_t)
// (c_t == 0: explicit fields only), default seeded weights.  The output
// matrix goes to out (capacity out_cap floats), dims to *rows / *cols.
int ref_run_network(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed,
                    const float* input, int in_layout, float* out, uint64_t out_cap,
                    uint32_t* rows, uint32_t* cols) {
  GUARD({
    R::NetworkSpec spec = R::parse_network(json);
    if (c_t) spec = R::annotate_layouts(spec, R::HeuristicThresholds{c_t, n_t});
    R::Tensor4D in(spec.n, spec.c, spec.h, spec.w, static_cast<R::Layout>(in_layout));
    std::copy(input, input + in.size(), in.data());
    R::RunOptions opt;
    opt.seed = seed;
    const R::RunResult res = R::run_network(spec, in, opt);
    const auto* m = std::get_if<R::Matrix>(&res.output);
    if (!m) throw std::runtime_error("ref_run_network: network does not end in a matrix");
    if (m->data.size() > out_cap) throw std::runtime_error("ref_run_network: output too large");
    *rows = m->rows;
    *cols = m->cols;
    std::copy(m->data.begin(), m->data.end(), out);
  })
}

// ref_run_network over `threads` std::threads, each running the unmodified
// run_network on its own N-shard of the input (NCHW input only: shards are
// contiguous image blocks) and writing its logits rows in image order.  Used
// to pin the full-size GPU forwards on a multi-image slice in seconds
// (batch independence, test_conv.cpp:117-141).
int ref_run_network_sharded(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed,
                            const float* input, uint32_t n, float* out, uint64_t out_cap,
                            uint32_t* rows, uint32_t* cols, int threads) {
  GUARD({
    if (threads < 1) threads = 1;
    if (static_cast<uint32_t>(threads) > n) threads = static_cast<int>(n);
    const R::NetworkSpec base_spec = R::parse_network(json);
    const uint64_t img = static_cast<uint64_t>(base_spec.c) * base_spec.h * base_spec.w;
    std::vector<std::string> errs(threads);
    std::vector<uint32_t> cls(threads, 0);
    auto work = [&](int t) {
      try {
        const uint32_t per = n / threads, extra = n % threads;
        const uint32_t a = t * per + std::min<uint32_t>(t, extra);
        const uint32_t b = a + per + (static_cast<uint32_t>(t) < extra ? 1 : 0);
        R::NetworkSpec spec = base_spec;
        spec.n = b - a;
        if (c_t) spec = R::annotate_layouts(spec, R::HeuristicThresholds{c_t, n_t});
        R::Tensor4D in(spec.n, spec.c, spec.h, spec.w, R::Layout::NCHW);
        std::copy(input + a * img, input + b * img, in.data());
        R::RunOptions opt;
        opt.seed = seed;
        const R::RunResult res = R::run_network(spec, in, opt);
        const auto* m = std::get_if<R::Matrix>(&res.output);
        if (!m) throw std::runtime_error("ref_run_network_sharded: output is not a matrix");
        if (static_cast<uint64_t>(b) * m->cols > out_cap)
          throw std::runtime_error("ref_run_network_sharded: output too large");
        cls[t] = m->cols;
        std::copy(m->data.begin(), m->data.end(), out + static_cast<uint64_t>(a) * m->cols);
      } catch (const std::exception& e) {
        errs[t] = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    *rows = n;
    *cols = cls[0];
  })
}

// fixture_list_csv (fixtures.cpp) -- the `lcnn fixtures --list` body
const char* ref_fixture_list_csv(uint32_t scale) {
  static std::string text;
  try {
    text = R::fixture_list_csv(scale);
  } catch (...) {
    map_current_exception();
    return nullptr;
  }
  return text.c_str();
}

// The `lcnn run-net CONFIG --preset P --seed S` body of the reference CLI
// (tools/lcnn.cpp:212-236): preset thresholds, annotation, a seeded input in
// the first 4D layer's layout, run_network, timing_report_csv.
const char* ref_run_net_cli(const char* json, const char* preset, uint64_t seed) {
  static std::string text;
  try {
    R::NetworkSpec spec = R::parse_network(json);
    const auto th = R::preset_by_name(preset);
    if (!th) throw R::ValidationError("unknown preset");
    spec = R::annotate_layouts(std::move(spec), *th);
    R::Layout first = R::Layout::NCHW;
    for (const R::LayerSpec& l : spec.layers)
      if ((l.kind == R::LayerKind::Convolution || l.kind == R::LayerKind::Pooling) && l.layout_field) {
        first = *l.layout_field;
        break;
      }
    R::Tensor4D in(spec.n, spec.c, spec.h, spec.w, first);
    std::mt19937 rng(static_cast<std::uint32_t>(seed));
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    for (std::uint64_t i = 0; i < in.size(); ++i) in.data()[i] = dist(rng);
    R::RunOptions opt;
    opt.seed = seed;
    text = R::timing_report_csv(R::run_network(spec, in, opt).report);
  } catch (...) {
    map_current_exception();
    return nullptr;
  }
  return text.c_str();
}

}  // extern "C"
