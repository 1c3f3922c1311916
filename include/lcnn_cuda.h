/*
 * lcnn_cuda.h -- C ABI of the B200 (sm_100a) memory-bound CNN layer path.
 *
 * This is the drop-in boundary between the reference's C++ operator API
 * (/root/reference/proj/include/lcnn/ headers) and hand-written CUDA kernels.
 * Every entry point takes caller-owned DEVICE pointers plus a cudaStream_t
 * (passed as void* so this header needs no CUDA include), validates its
 * parameters synchronously on the host with the reference's rules, and then
 * enqueues stream-ordered kernels.  Nothing here allocates or frees device
 * memory; nothing here synchronises the stream.
 *
 * Each entry cites the reference interface it replaces (file:line relative to
 * /root/reference/proj).  Errors map 1:1 onto the reference exception types
 * of include/lcnn/errors.hpp:8-56; the C++ host layer (host/include/lcnn/)
 * rethrows them with the same message text (lcnn_last_error()).
 *
 * Tensor layouts use the reference's codes (tensor.hpp:16): the last-named
 * dimension is contiguous.
 */
#ifndef LCNN_CUDA_H_
#define LCNN_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCNN_ABI_VERSION 1

/* Status codes; one per exception class of errors.hpp:8-56 plus CUDA/arg. */
typedef enum lcnn_status {
  LCNN_OK = 0,
  LCNN_ESHAPE = 1,        /* ShapeError        errors.hpp:13 */
  LCNN_EINDEX = 2,        /* IndexError        errors.hpp:18 */
  LCNN_ELAYOUT = 3,       /* LayoutError       errors.hpp:23 */
  LCNN_EPLAN = 4,         /* PlanError         errors.hpp:28 */
  LCNN_EFORMAT = 5,       /* FormatError       errors.hpp:33 */
  LCNN_EDOMAIN = 6,       /* DomainError       errors.hpp:38 */
  LCNN_EUNSUPPORTED = 7,  /* UnsupportedError  errors.hpp:43 */
  LCNN_EVALIDATION = 8,   /* ValidationError   errors.hpp:48 */
  LCNN_ECALIBRATION = 9,  /* CalibrationError  errors.hpp:53 */
  LCNN_ECUDA = 10,        /* CUDA runtime failure (launch, bad pointer) */
  LCNN_EINVAL = 11        /* null pointer / bad enum at the ABI level */
} lcnn_status;

/* Layout codes == lcnn::Layout (tensor.hpp:16) and the T4D1 layout byte. */
typedef enum lcnn_layout {
  LCNN_NCHW = 0,
  LCNN_CHWN = 1,
  LCNN_NHWC = 2,
  LCNN_HWCN = 3
} lcnn_layout;

/* == lcnn::PoolMode (pool.hpp:11). */
typedef enum lcnn_pool_mode { LCNN_POOL_MAX = 0, LCNN_POOL_AVG = 1 } lcnn_pool_mode;

/* == lcnn::AccessReport (pool.hpp:30-34).  Computed analytically on the host
 * with the reference's counting rules; the kernels themselves are measured
 * with ncu (dram__bytes_*). */
typedef struct lcnn_access_report {
  uint64_t input_loads;
  uint64_t output_stores;
  uint64_t distinct_inputs;
} lcnn_access_report;

/* == lcnn::PassReport (softmax.hpp:21-24). */
typedef struct lcnn_pass_report {
  uint32_t materializations;
  uint32_t full_matrix_sweeps;
} lcnn_pass_report;

/* ---- library ----------------------------------------------------------- */
int lcnn_abi_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* lcnn_last_error(void);
const char* lcnn_status_name(int status);
/* 1 if a CUDA device of compute capability 10.x is usable, else 0. */
int lcnn_device_ok(void);

/* ---- layout transform (layout.hpp:12-40, layout.cpp:72-144) ------------ */
/* == flattenable_pair (layout.cpp:72-75). */
int lcnn_flattenable_pair(int src_layout, int dst_layout);

/* == transform (layout.cpp:138-144): CHWN<->NCHW run as a 2D transpose
 * [C*H*W]x[N] <-> [N]x[C*H*W]; other pairs run the generic 4D permute;
 * src == dst is a copy.  Bit-exact (pure data movement).  src and dst must
 * not overlap. */
lcnn_status lcnn_transform(const float* src, float* dst, uint32_t n, uint32_t c,
                           uint32_t h, uint32_t w, int src_layout,
                           int dst_layout, void* stream);

/* == transform_tiled (layout.cpp:99-120) with validate_plan's PlanError rules
 * (layout.cpp:13-26): pair must flatten, tile a power of two in [8,128],
 * wide_copy requires n >= 64.  On the GPU the tile and wide flags are hints:
 * the kernel always moves 128-bit vectors where alignment allows. */
lcnn_status lcnn_transform_tiled(const float* src, float* dst, uint32_t n,
                                 uint32_t c, uint32_t h, uint32_t w,
                                 int src_layout, int dst_layout, uint32_t tile,
                                 int wide_copy, void* stream);

/* == transform_naive (layout.cpp:77-97): element-wise 4D permutation for any
 * layout pair (the generic kernel; no 2D flattening). */
lcnn_status lcnn_transform_naive(const float* src, float* dst, uint32_t n,
                                 uint32_t c, uint32_t h, uint32_t w,
                                 int src_layout, int dst_layout, void* stream);

/* ---- pooling (pool.hpp:36-65, pool.cpp:19-270) -------------------------- */
/* == pool_output_extents (pool.cpp:44-47) plus check_window (pool.cpp:19-26)
 * so a caller can size the output before launching. */
lcnn_status lcnn_pool_output_extents(uint32_t h, uint32_t w, uint32_t win_h,
                                     uint32_t win_w, uint32_t stride,
                                     uint32_t* h_out, uint32_t* w_out);

/* ---- pooling plan tuner (PAPER.md:227 autotuned coarsening, pool.cpp:272-331) --
 * The kernel plan of one pooling shape: the (fh, fw) output block each thread
 * computes with register reuse of overlapping windows, and for the NCHW
 * pipelined kernel the shared-memory ring (KB per slot, slots per CTA, CTAs
 * per SM; 0 = the shape's default).  Any plan gives the same output bits (tap
 * order is per output), so plans change speed only. */
typedef struct lcnn_pool_plan {
  uint32_t fh, fw;
  uint32_t ring_kb, ring_slots, ring_ctas;
  int tuned;  /* 1: measured by lcnn_pool_tune on this device */
  float us;   /* measured time of the plan, microseconds (0 if untuned) */
} lcnn_pool_plan;
/* Measure every specialised plan of the layout's kernel family on scratch
 * buffers of this shape (CUDA events on `stream`, median of 3 after a
 * warm-up; CHWN fh, fw in 1..4; NCHW fh 1..4, fw 1..2, then 7 ring shapes),
 * cache the fastest per (device, shape, window, mode) and return it.  A shape
 * already tuned returns the cached plan without measuring.  Synchronises
 * `stream`; allocates the shape's input + output transiently. */
lcnn_status lcnn_pool_tune(uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout,
                           uint32_t win_h, uint32_t win_w, uint32_t stride, int mode,
                           lcnn_pool_plan* plan, void* stream);
/* The cached tuned plan, else the static default (no measurement). */
lcnn_status lcnn_pool_plan_lookup(uint32_t n, uint32_t c, uint32_t h, uint32_t w, int layout,
                                  uint32_t win_h, uint32_t win_w, uint32_t stride, int mode,
                                  lcnn_pool_plan* plan);
/* Pool in CHWN or NCHW with an explicit plan; report = the coarsened access
 * report of (fh, fw) (pool.cpp:236). */
lcnn_status lcnn_pool_run_plan(const float* src, float* dst, uint32_t n, uint32_t c,
                               uint32_t h, uint32_t w, int layout, uint32_t win_h,
                               uint32_t win_w, uint32_t stride, int mode,
                               const lcnn_pool_plan* plan, lcnn_access_report* report,
                               void* stream);

/* == pool_layout (pool.cpp:172-176 -> pool_plain :98-163).  layout must be
 * CHWN or NCHW (LayoutError otherwise, pool.cpp:165); output keeps the input
 * layout.  Max: bit-exact with acc = (acc < v) ? v : acc from -inf in (y,x)
 * tap order.  Average: fp32 adds from 0.0f in (y,x) order, then CHWN
 * multiplies by 1.0f/(wh*ww) while NCHW divides by float(wh*ww), as the
 * reference does.  report may be NULL. */
lcnn_status lcnn_pool_layout(const float* src, float* dst, uint32_t n,
                             uint32_t c, uint32_t h, uint32_t w, int layout,
                             uint32_t win_h, uint32_t win_w, uint32_t stride,
                             int mode, lcnn_access_report* report,
                             void* stream);

/* == pool_coarsened (pool.cpp:178-270): CHWN only (LayoutError otherwise),
 * PlanError if fh or fw < 1 or fh*fw > 64 (kCoarseningCap, pool.hpp:28).
 * Each thread keeps an fh x fw block of outputs in registers and loads the
 * receptive-field union once.  report uses the union-count formula. */
lcnn_status lcnn_pool_coarsened(const float* src, float* dst, uint32_t n,
                                uint32_t c, uint32_t h, uint32_t w, int layout,
                                uint32_t win_h, uint32_t win_w, uint32_t stride,
                                int mode, uint32_t fh, uint32_t fw,
                                lcnn_access_report* report, void* stream);

/* GPU extension (not in the reference API, which rejects NCHW coarsening,
 * pool.cpp:189-191): the register-coarsened NCHW kernel.  Same output bits
 * as lcnn_pool_layout on NCHW; report counts the union loads. */
lcnn_status lcnn_pool_coarsened_nchw(const float* src, float* dst, uint32_t n,
                                     uint32_t c, uint32_t h, uint32_t w,
                                     uint32_t win_h, uint32_t win_w,
                                     uint32_t stride, int mode, uint32_t fh,
                                     uint32_t fw, lcnn_access_report* report,
                                     void* stream);

/* == pool_oracle (pool.cpp:49-84): any input layout, NCHW output, fp64
 * accumulation, max seeded from the first tap.  Ground truth, not a hot op. */
lcnn_status lcnn_pool_oracle(const float* src, float* dst, uint32_t n,
                             uint32_t c, uint32_t h, uint32_t w, int layout,
                             uint32_t win_h, uint32_t win_w, uint32_t stride,
                             int mode, void* stream);

/* ---- softmax (softmax.hpp:28-39, softmax.cpp:36-180) -------------------- */
/* == softmax_fused (softmax.cpp:100-180).  One kernel: the row is staged in
 * registers (or shared memory for wide rows), max and sum reduced with warp
 * shuffles + shared memory, no intermediate touches HBM.  Rows wider than
 * local_buffer_limit are reported as the streaming schedule (5 sweeps), as
 * the reference does.  d_nonfinite (device int, may be NULL) is zeroed on
 * the stream and set to 1 if any input is inf/NaN: the host wrapper reads it
 * and raises DomainError (softmax.cpp:15-19).  report may be NULL. */
lcnn_status lcnn_softmax_fused(const float* src, float* dst, uint32_t rows,
                               uint32_t cols, uint32_t local_buffer_limit,
                               int* d_nonfinite, lcnn_pass_report* report,
                               void* stream);
/* softmax_fused for a device-resident pipeline (the network executor's
 * classifier): the same kernel, but d_sticky (device int, may be NULL) is
 * never cleared -- it is set to 1 on a non-finite input and keeps that value
 * until the owner clears it, so an asynchronous forward needs no extra
 * zeroing launch and no host read (lcnn_net_status reads it). */
lcnn_status lcnn_softmax_fused_sticky(const float* src, float* dst, uint32_t rows,
                                      uint32_t cols, int* d_sticky, void* stream);

/* Device scratch (bytes) the five-pass path needs for (rows, cols). */
size_t lcnn_softmax_reference_scratch_bytes(uint32_t rows, uint32_t cols);

/* == softmax_reference (softmax.cpp:36-98): five kernels (max, subtract,
 * exp, blocked sum, normalise) each materialising its intermediate in the
 * caller's scratch -- the paper's multi-kernel baseline. */
lcnn_status lcnn_softmax_reference(const float* src, float* dst,
                                   uint32_t rows, uint32_t cols,
                                   void* d_scratch, size_t scratch_bytes,
                                   int* d_nonfinite, lcnn_pass_report* report,
                                   void* stream);

/* ---- convolution / fully-connected (conv.hpp:17-54, softmax.cpp:182) ---- */
/* == conv_output_extents (conv.cpp:22-33). */
lcnn_status lcnn_conv_output_extents(uint32_t h, uint32_t w, uint32_t f_h,
                                     uint32_t f_w, uint32_t stride,
                                     uint32_t pad, uint32_t* h_out,
                                     uint32_t* w_out);

/* Arithmetic of the dense paths. */
typedef enum lcnn_precision {
  LCNN_PREC_TF32 = 0,   /* tcgen05 kind::tf32, one MMA chain (fastest)       */
  LCNN_PREC_3XTF32 = 1, /* tcgen05, hi*hi + hi*lo + lo*hi: ~fp32 accuracy    */
  LCNN_PREC_FP32 = 2    /* CUDA-core FFMA: fp32 products, fp32 accumulation  */
} lcnn_precision;

/* Bytes of device workspace lcnn_conv_forward needs (packed filters, and the
 * split operand copies in 3xTF32 mode). */
size_t lcnn_conv_workspace_bytes(uint32_t n, uint32_t c_i, uint32_t h,
                                 uint32_t w, uint32_t c_o, uint32_t f_h,
                                 uint32_t f_w, int precision);
/* Workspace of lcnn_conv_forward for this exact geometry (stride, padding,
 * layout): what the routed kernel needs.  The stride-free query above returns
 * a bound over every stride / padding. */
size_t lcnn_conv_workspace_bytes_ex(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                    int layout, uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                    uint32_t stride, uint32_t pad, int precision);

/* == conv_direct (conv.cpp:200-213) and conv_gemm (conv.cpp:306-332): the
 * convolution of an (n, c_i, h, w) input in CHWN or NCHW (LayoutError
 * otherwise), output (n, c_o, h_out, w_out) in the input's layout.  filters
 * are (c_o, c_i, f_h, f_w) (tensor.hpp:77-103).  CHWN with n % 32 == 0 runs
 * the implicit-GEMM tcgen05 kernel (TF32 / 3xTF32); FP32 precision and the
 * remaining shapes run the fp32 CUDA-core kernel. */
lcnn_status lcnn_conv_forward(const float* src, const float* filters,
                              float* dst, uint32_t n, uint32_t c_i, uint32_t h,
                              uint32_t w, int layout, uint32_t c_o,
                              uint32_t f_h, uint32_t f_w, uint32_t stride,
                              uint32_t pad, int precision, void* d_workspace,
                              size_t workspace_bytes, void* stream);

/* Filter pre-packing for convolutions whose weights are reused (network
 * layers; run_network re-reads the same FilterBank every forward,
 * net.cpp:284-330): lcnn_conv_forward split into its two phases.  A packed
 * image is the operand layout of the kernel the geometry + precision route
 * to, valid only for that exact (n, c_i, h, w, layout, c_o, f_h, f_w,
 * stride, pad, precision); d_packed must be 256-byte aligned.  Sizes return
 * 0 for invalid geometry.  lcnn_conv_forward_packed == lcnn_conv_forward on
 * the filters that were packed, bit for bit. */
size_t lcnn_conv_packed_bytes(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                              int layout, uint32_t c_o, uint32_t f_h,
                              uint32_t f_w, uint32_t stride, uint32_t pad,
                              int precision);
size_t lcnn_conv_packed_workspace_bytes(uint32_t n, uint32_t c_i, uint32_t h,
                                        uint32_t w, int layout, uint32_t c_o,
                                        uint32_t f_h, uint32_t f_w,
                                        uint32_t stride, uint32_t pad,
                                        int precision);
lcnn_status lcnn_conv_pack_filters(const float* filters, void* d_packed,
                                   size_t packed_bytes, uint32_t n,
                                   uint32_t c_i, uint32_t h, uint32_t w,
                                   int layout, uint32_t c_o, uint32_t f_h,
                                   uint32_t f_w, uint32_t stride, uint32_t pad,
                                   int precision, void* stream);
lcnn_status lcnn_conv_forward_packed(const float* src, const void* d_packed,
                                     float* dst, uint32_t n, uint32_t c_i,
                                     uint32_t h, uint32_t w, int layout,
                                     uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                     uint32_t stride, uint32_t pad,
                                     int precision, void* d_workspace,
                                     size_t workspace_bytes, void* stream);

/* lcnn_conv_forward_packed with caller-owned SYNC WORDS: d_sync is NULL
 * (== lcnn_conv_forward_packed) or LCNN_SYNC_BYTES of 8-byte-aligned device
 * memory, zero before its first use, that belongs to ONE call site (e.g. one
 * network layer on one stream) whose launches never overlap in time.  A
 * persistent tensor-core kernel whose stream-K tail adds fragments into the
 * output then zeroes that output region itself, overlapped with its operand
 * loads, instead of needing a separate zeroing launch ahead of it; the
 * kernel leaves the words zero again.  Results are those of
 * lcnn_conv_forward_packed. */
#define LCNN_SYNC_BYTES 16
lcnn_status lcnn_conv_forward_packed_ex(const float* src, const void* d_packed,
                                        float* dst, uint32_t n, uint32_t c_i,
                                        uint32_t h, uint32_t w, int layout,
                                        uint32_t c_o, uint32_t f_h,
                                        uint32_t f_w, uint32_t stride,
                                        uint32_t pad, int precision,
                                        void* d_workspace,
                                        size_t workspace_bytes, void* d_sync,
                                        void* stream);

/* Convolution followed by max pooling as ONE kernel (the run_network layer
 * pair conv -> pool, net.cpp:284-353, when the pool consumes the conv output
 * in the same layout): the conv output never reaches HBM.  Supported for
 * CHWN, TF32, layers the SHARE route takes (small c_i * f_w, c_o <= 128,
 * e.g. AlexNet conv1) with square max windows of 2 or 3 at stride 2, and
 * layers the TAPS route takes at stride 1 (c_i % 32 == 0, channel planes
 * >= 4 MB, e.g. VGG-16 conv1_2, conv2_2) with a 2 x 2 window at stride 2.
 * d_packed is the layer's lcnn_conv_pack_filters image (same geometry and
 * precision); dst receives the (n, c_o, hp, wp) CHWN pooled output,
 * hp/wp = pool_output_extents of the conv output.  Bit-identical to
 * lcnn_conv_forward_packed followed by lcnn_pool_layout (max).
 * lcnn_conv_maxpool_supported returns 1 when the fused kernel covers the
 * geometry, 0 otherwise (callers then run the two layers). */
int lcnn_conv_maxpool_supported(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                                int layout, uint32_t c_o, uint32_t f_h,
                                uint32_t f_w, uint32_t stride, uint32_t pad,
                                int precision, uint32_t pool_win,
                                uint32_t pool_stride);
lcnn_status lcnn_conv_maxpool_packed(const float* src, const void* d_packed,
                                     float* dst, uint32_t n, uint32_t c_i,
                                     uint32_t h, uint32_t w, int layout,
                                     uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                     uint32_t stride, uint32_t pad,
                                     int precision, uint32_t pool_win,
                                     uint32_t pool_stride, void* stream);

/* Blocked activation layout between two convolutions inside run_network (not
 * a reference layout; never crosses the API): [N/32][H][W][C][32].  A TAPS
 * row-pair convolution reads its input boxes from it as runs of 4 KB instead
 * of 128-B lines of 32 channel planes (VGG conv1_2 + pool1 1.42 -> 0.93 ms,
 * profiles/r02_tma_bench_blocked_layouts.txt); the ROW row-pair producer
 * writes it through its quad-box epilogue.  Flags of the two _blk calls: */
#define LCNN_CONV_IN_HWCN32 1u  /* src is blocked (conv_maxpool, TAPS row pairs) */
#define LCNN_CONV_OUT_HWCN32 2u /* dst is blocked (conv_forward, ROW row pairs) */
/* 1 when the route of this CHWN geometry reads / writes the blocked layout the
 * flags name (pool_win = 0: plain conv) */
int lcnn_conv_hwcn32_supported(uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                               uint32_t c_o, uint32_t f_h, uint32_t f_w,
                               uint32_t stride, uint32_t pad, int precision,
                               uint32_t pool_win, uint32_t pool_stride,
                               uint32_t flags);
lcnn_status lcnn_conv_forward_packed_blk(const float* src, const void* d_packed,
                                         float* dst, uint32_t n, uint32_t c_i,
                                         uint32_t h, uint32_t w, int layout,
                                         uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                         uint32_t stride, uint32_t pad,
                                         int precision, void* d_workspace,
                                         size_t workspace_bytes, void* d_sync,
                                         uint32_t flags, void* stream);
lcnn_status lcnn_conv_maxpool_packed_blk(const float* src, const void* d_packed,
                                         float* dst, uint32_t n, uint32_t c_i,
                                         uint32_t h, uint32_t w, int layout,
                                         uint32_t c_o, uint32_t f_h, uint32_t f_w,
                                         uint32_t stride, uint32_t pad,
                                         int precision, uint32_t pool_win,
                                         uint32_t pool_stride, uint32_t flags,
                                         void* stream);

/* == conv_oracle (conv.cpp:53-93): fp64 accumulation, any input layout,
 * NCHW output.  Ground truth, not a hot op. */
lcnn_status lcnn_conv_oracle(const float* src, const float* filters, float* dst,
                             uint32_t n, uint32_t c_i, uint32_t h, uint32_t w,
                             int layout, uint32_t c_o, uint32_t f_h,
                             uint32_t f_w, uint32_t stride, uint32_t pad,
                             void* stream);

/* == im2col (conv.cpp:215-250): NCHW input (LayoutError otherwise) unrolled
 * to a (c_i*f_h*f_w) x (n*h_out*w_out) row-major matrix, padded taps 0. */
lcnn_status lcnn_im2col(const float* src, float* dst, uint32_t n, uint32_t c_i,
                        uint32_t h, uint32_t w, int layout, uint32_t f_h,
                        uint32_t f_w, uint32_t stride, uint32_t pad,
                        void* stream);

/* Bytes of device workspace lcnn_gemm needs (0 unless 3xTF32). */
size_t lcnn_gemm_workspace_bytes(uint64_t m, uint64_t n, uint64_t k,
                                 int precision);

/* == gemm_blocked (conv.cpp:252-304) / fc_forward (softmax.cpp:182-184):
 * c (m x n) = a (m x k) * b (k x n), all row-major fp32.  TF32 / 3xTF32 run
 * the tcgen05 kernel when k and n are multiples of 4 (TMA pitch rule), else
 * the fp32 CUDA-core kernel. */
lcnn_status lcnn_gemm(const float* a, const float* b, float* c, uint64_t m,
                      uint64_t n, uint64_t k, int precision, void* d_workspace,
                      size_t workspace_bytes, void* stream);

/* fc_forward (softmax.cpp:182-184) with weights that are reused across calls
 * (network fc layers; run_network re-reads the same weights every forward,
 * net.cpp:338-383): the weights (k x n, row-major) are packed ONCE into the
 * tensor-core operand image (W^T, K-major; + the 3xTF32 split), then
 * y (m x n) = x . W runs on it.  x_layout LCNN_NCHW: x is m rows of k
 * (the flattened NCHW activations); LCNN_CHWN: x is the CHWN producer itself,
 * [k][m] with the m images contiguous, so the flatten (net.cpp:258-262) costs
 * no transform.  TF32 / 3xTF32 only (packed_bytes 0 otherwise); k % 4 == 0,
 * and m % 4 == 0 for CHWN.  d_packed 256-byte aligned. */
size_t lcnn_fc_packed_bytes(uint64_t k, uint64_t n, int precision);
size_t lcnn_fc_workspace_bytes(uint64_t m, uint64_t k, int precision);
lcnn_status lcnn_fc_pack_weights(const float* weights, void* d_packed,
                                 size_t packed_bytes, uint64_t k, uint64_t n,
                                 int precision, void* stream);
lcnn_status lcnn_fc_forward_packed(const float* x, int x_layout,
                                   const void* d_packed, float* y, uint64_t m,
                                   uint64_t n, uint64_t k, int precision,
                                   void* d_workspace, size_t workspace_bytes,
                                   void* stream);
/* lcnn_fc_forward_packed with caller-owned sync words (d_sync: see
 * lcnn_conv_forward_packed_ex): the stream-K output is zeroed inside the fc
 * kernel instead of by a separate launch.  d_next_packed / next_bytes
 * (optional, NULL / 0): the NEXT fc layer's packed weights; once a CTA has
 * issued its own loads it prefetches its share of them into L2, so the next
 * layer starts on L2 hits while this one drains (weights never depend on
 * this layer's output). */
lcnn_status lcnn_fc_forward_packed_ex(const float* x, int x_layout,
                                      const void* d_packed, float* y,
                                      uint64_t m, uint64_t n, uint64_t k,
                                      int precision, void* d_workspace,
                                      size_t workspace_bytes, void* d_sync,
                                      const void* d_next_packed,
                                      size_t next_bytes, void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* LCNN_CUDA_H_ */
