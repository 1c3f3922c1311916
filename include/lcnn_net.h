/*
 * lcnn_net.h -- C ABI of the network runtime (liblcnn.so), the B200 form of
 * the reference's run_network / annotate_layouts / plan_transforms
 * (proj/include/lcnn/net.hpp:58-131).  A handle owns the parsed, annotated
 * network and its weights resident in HBM; forward runs on a caller stream
 * with device buffers (value) or host buffers (end to end).
 */
#ifndef LCNN_NET_H_
#define LCNN_NET_H_

#include <stddef.h>
#include <stdint.h>

#include "lcnn_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lcnn_net lcnn_net;

/* parse_network (net.cpp:51-118) + annotate_layouts (net.cpp:186-195) with
 * thresholds (c_t, n_t) for layers whose layout is "auto" (c_t == 0 selects
 * the titan-black preset), weights from the reference's seeded streams
 * (net.cpp:217-243) uploaded once.  Returns an lcnn_status. */
int lcnn_net_create(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed,
                    lcnn_net** out);
/* lcnn_net_create with the conv / fc precision (lcnn_precision; -1 = the
 * process default of lcnn_set_dense_precision at this call).  The precision
 * is fixed per network: networks at different precisions may run
 * concurrently on different threads.  Filters and fc weights are packed for
 * their layer's kernel here, once. */
int lcnn_net_create_ex(const char* json, uint32_t c_t, uint32_t n_t, uint64_t seed,
                       int precision, lcnn_net** out);
/* The network's lcnn_precision. */
int lcnn_net_precision(const lcnn_net* net);
/* The GPU-tuned pooling plan of layer `layer` (lcnn_pool_tune, measured when
 * the network was created; tuned == 0 for non-pool layers). */
int lcnn_net_pool_plan(const lcnn_net* net, uint32_t layer, lcnn_pool_plan* plan);
void lcnn_net_destroy(lcnn_net* net);
const char* lcnn_net_last_error(void);

/* Input dims, the layout the first 4D layer consumes, output matrix dims,
 * forward flops per image, transforms executed for an input in in_layout. */
int lcnn_net_info(const lcnn_net* net, int in_layout, uint32_t dims[4],
                  int* first_layout, uint32_t* out_rows, uint32_t* out_cols,
                  uint64_t* flops_per_image, uint32_t* transforms);
/* Per-layer layout codes after annotation (-1 for fc/softmax). */
int lcnn_net_layouts(const lcnn_net* net, int* layouts, uint32_t max_layers);

/* Forward with device buffers on `stream` (a cudaStream_t).  Asynchronous:
 * a non-finite classifier input (the reference's DomainError,
 * softmax.cpp:15-19) sets the network's sticky device flag instead of
 * blocking; lcnn_net_status reports it. */
int lcnn_net_forward(const lcnn_net* net, const float* d_input, int in_layout,
                     float* d_output, void* stream);
/* lcnn_net_forward replayed from a CUDA graph: the first call for a given
 * (d_input, in_layout, d_output) captures one whole forward -- every layer,
 * inserted transform and the classifier -- into a graph owned by the
 * network (at most 16 cached; the oldest is dropped after a device sync);
 * later calls with the same buffers are one cudaGraphLaunch on `stream`.
 * Same results and non-finite-flag semantics as lcnn_net_forward.  Replays
 * of one cached graph are serialised by CUDA; the buffers must stay valid
 * while the network lives. */
int lcnn_net_forward_graph(lcnn_net* net, const float* d_input, int in_layout,
                           float* d_output, void* stream);
/* Wait for `stream`, read and clear the non-finite flag: LCNN_EDOMAIN
 * ("layer '<softmax>': softmax: non-finite input") if any forward since the
 * last call met a non-finite input, else LCNN_OK. */
int lcnn_net_status(const lcnn_net* net, void* stream);
/* The sticky flag itself (device int, 0 or 1) for callers that poll it on
 * the device or copy it back themselves; clear it with cudaMemsetAsync. */
const int* lcnn_net_nonfinite_flag(const lcnn_net* net);
/* Forward with host buffers: H2D, forward, D2H (synchronous); returns
 * LCNN_EDOMAIN for a non-finite classifier input. */
int lcnn_net_forward_host(const lcnn_net* net, const float* h_input,
                          int in_layout, float* h_output);
/* `count` forwards over host buffers h_inputs[i] -> h_outputs[i] (pinned
 * memory for overlap), pipelined: the H2D of batch i+1 runs on a copy stream
 * into the other of two device input buffers while batch i computes; each
 * result is read back (D2H) on the compute stream.  Returns when every output
 * has landed.  The streaming form of run_network's host-buffer contract
 * (net.cpp:266-398) for a sequence of batches. */
int lcnn_net_forward_host_many(const lcnn_net* net, const float* const* h_inputs,
                               int in_layout, float* const* h_outputs, uint32_t count);

/* One forward with per-entry CUDA-event device times (layers and inserted
 * transforms, in execution order): nanos[i], names comma-separated. */
int lcnn_net_profile(const lcnn_net* net, const float* d_input, int in_layout,
                     void* stream, uint64_t* nanos, uint32_t max_entries,
                     char* names, size_t names_len, uint32_t* count);

/* Process default lcnn_precision for networks created afterwards with
 * lcnn_net_create (FP32 unless LCNN_DENSE_PRECISION says otherwise) and for
 * the host-tensor conv / fc calls. */
void lcnn_set_dense_precision(int precision);

#ifdef __cplusplus
}
#endif

#endif /* LCNN_NET_H_ */
