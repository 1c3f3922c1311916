// C ABI of the network runtime (include/lcnn_net.h).
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>

#include "lcnn/net.hpp"
#include "lcnn_cuda.h"
#include "lcnn_net.h"

// Cached CUDA graphs of whole forwards (lcnn_net_forward_graph), one per
// (input, layout, output) buffer triple: a replay is one cudaGraphLaunch
// instead of the executor's ~11-30 launches and tensor-map encodes.
struct NetGraphs {
  using Key = std::tuple<const void*, int, void*>;
  static constexpr std::size_t kMax = 16;
  std::mutex mu;
  cudaStream_t capture = nullptr;  // private stream the forwards are captured on
  std::map<Key, cudaGraphExec_t> execs;
  std::map<Key, cudaGraph_t> graphs;
  ~NetGraphs() {
    for (auto& kv : execs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : graphs) cudaGraphDestroy(kv.second);
    if (capture) cudaStreamDestroy(capture);
  }
};

struct lcnn_net {
  std::unique_ptr<lcnn::Network> net;
  NetGraphs graphs;
};

namespace {

thread_local std::string g_err;

int status_of_current() {
  try {
    throw;
  } catch (const lcnn::ShapeError& e) {
    g_err = e.what();
    return LCNN_ESHAPE;
  } catch (const lcnn::LayoutError& e) {
    g_err = e.what();
    return LCNN_ELAYOUT;
  } catch (const lcnn::PlanError& e) {
    g_err = e.what();
    return LCNN_EPLAN;
  } catch (const lcnn::DomainError& e) {
    g_err = e.what();
    return LCNN_EDOMAIN;
  } catch (const lcnn::UnsupportedError& e) {
    g_err = e.what();
    return LCNN_EUNSUPPORTED;
  } catch (const lcnn::ValidationError& e) {
    g_err = e.what();
    return LCNN_EVALIDATION;
  } catch (const lcnn::Error& e) {
    g_err = e.what();
    return LCNN_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LCNN_EINVAL;
  }
}

#define NET_GUARD(...)            \
  try {                           \
    __VA_ARGS__;                  \
    g_err.clear();                \
    return LCNN_OK;               \
  } catch (...) {                 \
    return status_of_current();   \
  }

lcnn::Layout L(int code) { return static_cast<lcnn::Layout>(code); }

// DomainError for a forward that met a non-finite classifier input, with the
// reference's layer-prefixed message (softmax.cpp:15-19 rethrown by
// net.cpp:387-391 as "layer '<name>': softmax: non-finite input").
void raise_if_nonfinite(const lcnn::Network& net) {
  if (net.take_nonfinite())
    throw lcnn::DomainError("layer '" + net.softmax_layer() + "': softmax: non-finite input");
}

// The ABI's stream argument is a cudaStream_t: 0 is the legacy default
// stream (CUDA's convention), not the library's private stream.
void* abi_stream(void* stream) { return stream ? stream : static_cast<void*>(cudaStreamLegacy); }

}  // namespace

extern "C" {

const char* lcnn_net_last_error(void) { return g_err.c_str(); }

void lcnn_set_dense_precision(int precision) { lcnn::set_dense_precision(precision); }

int lcnn_net_create_ex(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed,
                       int precision, lcnn_net** out) {
  NET_GUARD({
    if (!out) throw lcnn::ValidationError("null handle pointer");
    if (precision > LCNN_PREC_FP32) throw lcnn::ValidationError("unknown precision");
    lcnn::NetworkSpec spec = lcnn::parse_network(json);
    lcnn::HeuristicThresholds th = c_t ? lcnn::HeuristicThresholds{c_t, n_t} : lcnn::kTitanBlack;
    spec = lcnn::annotate_layouts(spec, th);
    lcnn::RunOptions opt;
    opt.seed = seed;
    opt.dense_precision = precision;
    auto* h = new lcnn_net{std::make_unique<lcnn::Network>(std::move(spec), opt)};
    *out = h;
  })
}

int lcnn_net_create(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed, lcnn_net** out) {
  return lcnn_net_create_ex(json, c_t, n_t, seed, -1, out);
}

int lcnn_net_precision(const lcnn_net* net) { return net->net->precision(); }

int lcnn_net_pool_plan(const lcnn_net* net, uint32_t layer, lcnn_pool_plan* plan) {
  NET_GUARD({
    if (!plan) throw lcnn::ValidationError("null plan pointer");
    if (layer >= net->net->spec().layers.size()) throw lcnn::ValidationError("layer out of range");
    *plan = net->net->pool_plan(layer);
  })
}

const int* lcnn_net_nonfinite_flag(const lcnn_net* net) { return net->net->nonfinite_flag(); }

int lcnn_net_status(const lcnn_net* net, void* stream) {
  NET_GUARD({
    lcnn::set_current_stream(abi_stream(stream));
    raise_if_nonfinite(*net->net);
  })
}

void lcnn_net_destroy(lcnn_net* net) { delete net; }

int lcnn_net_info(const lcnn_net* net, int in_layout, uint32_t dims[4], int* first_layout,
                  uint32_t* out_rows, uint32_t* out_cols, uint64_t* flops_per_image,
                  uint32_t* transforms) {
  NET_GUARD({
    const lcnn::NetworkSpec& s = net->net->spec();
    dims[0] = s.n;
    dims[1] = s.c;
    dims[2] = s.h;
    dims[3] = s.w;
    *first_layout = static_cast<int>(net->net->input_layout());
    const auto shapes = lcnn::infer_shapes(s);
    const lcnn::StageShape& o = shapes.back();
    *out_rows = o.n;
    *out_cols = o.c * o.h * o.w;
    *flops_per_image = net->net->flops_per_image();
    *transforms = static_cast<uint32_t>(net->net->transform_count(L(in_layout)));
  })
}

int lcnn_net_layouts(const lcnn_net* net, int* layouts, uint32_t max_layers) {
  NET_GUARD({
    const auto& layers = net->net->spec().layers;
    for (uint32_t i = 0; i < max_layers && i < layers.size(); ++i)
      layouts[i] = layers[i].layout_field ? static_cast<int>(*layers[i].layout_field) : -1;
  })
}

int lcnn_net_forward(const lcnn_net* net, const float* d_input, int in_layout, float* d_output,
                     void* stream) {
  NET_GUARD({
    lcnn::set_current_stream(abi_stream(stream));
    const lcnn::NetworkSpec& s = net->net->spec();
    const lcnn::DeviceTensor4D in = lcnn::DeviceTensor4D::wrap(const_cast<float*>(d_input), s.n,
                                                               s.c, s.h, s.w, L(in_layout));
    // a network ending in softmax writes d_output directly (no copy node
    // between forwards, which would also break the PDL chain)
    const lcnn::DeviceMatrix out = net->net->forward(in, nullptr, d_output);
    if (out.data() != d_output) {
      const cudaError_t e =
          cudaMemcpyAsync(d_output, out.data(), std::size_t{out.rows} * out.cols * sizeof(float),
                          cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
    }
  })
}

int lcnn_net_forward_graph(lcnn_net* net, const float* d_input, int in_layout, float* d_output,
                           void* stream) {
  NET_GUARD({
    if (!net) throw lcnn::ValidationError("null network");
    NetGraphs& g = net->graphs;
    const NetGraphs::Key key{d_input, in_layout, d_output};
    cudaGraphExec_t exec = nullptr;
    std::lock_guard<std::mutex> lock(g.mu);  // held through a capture (rare) and the launch
    const auto it = g.execs.find(key);
    if (it != g.execs.end()) exec = it->second;
    if (!exec) {
      // capture one forward on a private stream (nothing executes during a
      // capture, so the caller's stream needs no ordering against it), then
      // instantiate; allocations become graph memory nodes, the stream-K
      // sync words are a set of the capture's own (Network::sync_words)
      if (!g.capture) {
        const cudaError_t e = cudaStreamCreateWithFlags(&g.capture, cudaStreamNonBlocking);
        if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
      }
      cudaError_t e = cudaStreamBeginCapture(g.capture, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
      cudaGraph_t graph = nullptr;
      void* const prev = lcnn::current_stream();
      struct Restore {
        void* s;
        ~Restore() { lcnn::set_current_stream(s); }
      } restore{prev};
      try {
        lcnn::set_current_stream(g.capture);
        const lcnn::NetworkSpec& sp = net->net->spec();
        const lcnn::DeviceTensor4D in = lcnn::DeviceTensor4D::wrap(
            const_cast<float*>(d_input), sp.n, sp.c, sp.h, sp.w, L(in_layout));
        const lcnn::DeviceMatrix out = net->net->forward(in, nullptr, d_output);
        if (out.data() != d_output) {
          e = cudaMemcpyAsync(d_output, out.data(), std::size_t{out.rows} * out.cols * sizeof(float),
                              cudaMemcpyDeviceToDevice, g.capture);
          if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
        }
      } catch (...) {
        cudaStreamEndCapture(g.capture, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      e = cudaStreamEndCapture(g.capture, &graph);
      if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
      e = cudaGraphInstantiate(&exec, graph, 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        throw lcnn::Error(cudaGetErrorString(e));
      }
      if (g.execs.size() >= NetGraphs::kMax) {  // bounded cache: drop one entry
        auto victim = g.execs.begin();
        cudaStreamSynchronize(g.capture);
        cudaDeviceSynchronize();  // its last replay may still run
        cudaGraphExecDestroy(victim->second);
        cudaGraphDestroy(g.graphs[victim->first]);
        g.graphs.erase(victim->first);
        g.execs.erase(victim);
      }
      g.execs[key] = exec;
      g.graphs[key] = graph;
    }
    // launched under the lock: an eviction by another thread cannot destroy
    // the executable between the lookup and the launch
    const cudaError_t e = cudaGraphLaunch(exec, static_cast<cudaStream_t>(abi_stream(stream)));
    if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
  })
}

int lcnn_net_forward_host(const lcnn_net* net, const float* h_input, int in_layout,
                          float* h_output) {
  NET_GUARD({
    lcnn::set_current_stream(nullptr);
    const lcnn::NetworkSpec& s = net->net->spec();
    cudaStream_t st = static_cast<cudaStream_t>(lcnn::current_stream());
    lcnn::DeviceTensor4D in(s.n, s.c, s.h, s.w, L(in_layout));
    cudaError_t e = cudaMemcpyAsync(in.data(), h_input, in.size() * sizeof(float),
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
    const lcnn::DeviceMatrix out = net->net->forward(in);
    e = cudaMemcpyAsync(h_output, out.data(), std::size_t{out.rows} * out.cols * sizeof(float),
                        cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
    lcnn::synchronize();
    raise_if_nonfinite(*net->net);
  })
}

int lcnn_net_forward_host_many(const lcnn_net* net, const float* const* h_inputs, int in_layout,
                               float* const* h_outputs, uint32_t count) {
  struct Streams {  // copy stream + per-slot events, released on every exit path
    cudaStream_t copy = nullptr;
    cudaEvent_t loaded[2] = {}, consumed[2] = {};
    ~Streams() {
      // drain the copy stream before the input slots (declared earlier, so
      // destroyed later) go back to the allocator -- also on an error exit
      if (copy) cudaStreamSynchronize(copy);
      for (int b = 0; b < 2; ++b) {
        if (loaded[b]) cudaEventDestroy(loaded[b]);
        if (consumed[b]) cudaEventDestroy(consumed[b]);
      }
      if (copy) cudaStreamDestroy(copy);
    }
  };
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) throw lcnn::Error(cudaGetErrorString(e));
  };
  NET_GUARD({
    if (count && (!h_inputs || !h_outputs)) throw lcnn::ValidationError("null buffer array");
    lcnn::set_current_stream(nullptr);
    const lcnn::NetworkSpec& s = net->net->spec();
    cudaStream_t st = static_cast<cudaStream_t>(lcnn::current_stream());
    lcnn::DeviceTensor4D in[2] = {lcnn::DeviceTensor4D(s.n, s.c, s.h, s.w, L(in_layout)),
                                  lcnn::DeviceTensor4D(s.n, s.c, s.h, s.w, L(in_layout))};
    Streams r;
    ck(cudaStreamCreateWithFlags(&r.copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      ck(cudaEventCreateWithFlags(&r.loaded[b], cudaEventDisableTiming));
      ck(cudaEventCreateWithFlags(&r.consumed[b], cudaEventDisableTiming));
    }
    // the slots were allocated on the compute stream: the copy stream waits
    // for that before its first write
    for (int b = 0; b < 2; ++b) {
      ck(cudaEventRecord(r.consumed[b], st));
      ck(cudaStreamWaitEvent(r.copy, r.consumed[b], 0));
    }
    const std::size_t in_bytes = in[0].size() * sizeof(float);
    for (uint32_t i = 0; i < count; ++i) {
      const int b = static_cast<int>(i & 1);
      ck(cudaStreamWaitEvent(r.copy, r.consumed[b], 0));  // forward i-2 is done with slot b
      ck(cudaMemcpyAsync(in[b].data(), h_inputs[i], in_bytes, cudaMemcpyHostToDevice, r.copy));
      ck(cudaEventRecord(r.loaded[b], r.copy));
      ck(cudaStreamWaitEvent(st, r.loaded[b], 0));
      const lcnn::DeviceMatrix out = net->net->forward(in[b]);
      ck(cudaEventRecord(r.consumed[b], st));
      ck(cudaMemcpyAsync(h_outputs[i], out.data(), std::size_t{out.rows} * out.cols * sizeof(float),
                         cudaMemcpyDeviceToHost, st));
    }
    lcnn::synchronize();
    ck(cudaStreamSynchronize(r.copy));
    raise_if_nonfinite(*net->net);
  })
}

int lcnn_net_profile(const lcnn_net* net, const float* d_input, int in_layout, void* stream,
                     uint64_t* nanos, uint32_t max_entries, char* names, size_t names_len,
                     uint32_t* count) {
  NET_GUARD({
    lcnn::set_current_stream(abi_stream(stream));
    const lcnn::NetworkSpec& s = net->net->spec();
    const lcnn::DeviceTensor4D in = lcnn::DeviceTensor4D::wrap(const_cast<float*>(d_input), s.n,
                                                               s.c, s.h, s.w, L(in_layout));
    lcnn::TimingReport rep;
    (void)net->net->forward(in, &rep);
    std::string joined;
    uint32_t k = 0;
    for (const lcnn::LayerTiming& e : rep.entries) {
      if (k < max_entries) nanos[k] = e.nanos;
      ++k;
      if (!joined.empty()) joined += ',';
      joined += e.name;
    }
    *count = k;
    if (names && names_len) {
      std::strncpy(names, joined.c_str(), names_len - 1);
      names[names_len - 1] = 0;
    }
  })
}

}  // extern "C"
