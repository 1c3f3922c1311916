// Host-side launcher interface between the C ABI (capi.cu) and the kernel
// translation units.  Launchers assume validated parameters and return the
// cudaError_t of the launch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lcnn_impl {

// --- transform.cu -------------------------------------------------------
// dst[C][R] = transpose(src[R][C]), both row-major fp32.
cudaError_t launch_transpose2d(const float* src, float* dst, uint64_t rows,
                               uint64_t cols, cudaStream_t s);
// Generic 4D permutation between any two of the four layout codes.
cudaError_t launch_permute4d(const float* src, float* dst, uint32_t n,
                             uint32_t c, uint32_t h, uint32_t w, int src_layout,
                             int dst_layout, cudaStream_t s);

// --- pool.cu ------------------------------------------------------------
struct PoolArgs {
  const float* src;
  float* dst;
  uint32_t n, c, h, w;      // logical input extents
  uint32_t ho, wo;          // output extents
  uint32_t win_h, win_w, stride;
  bool avg;
  uint32_t fh, fw;          // coarsening factors (1,1 = plain kernel)
  // NCHW pipelined kernel's shared-memory ring: KB per slot, slots per CTA,
  // CTAs per SM (0 = the measured default for the shape)
  uint32_t ring_kb = 0, ring_slots = 0, ring_ctas = 0;
};
cudaError_t launch_pool_chwn(const PoolArgs& a, cudaStream_t s);
cudaError_t launch_pool_nchw(const PoolArgs& a, cudaStream_t s);
// fp64 oracle kernel: any layout in (strides in elements), NCHW out.
cudaError_t launch_pool_oracle(const PoolArgs& a, uint64_t sn, uint64_t sc,
                               uint64_t sh, uint64_t sw, cudaStream_t s);

// --- softmax.cu ---------------------------------------------------------
cudaError_t launch_softmax_fused(const float* src, float* dst, uint32_t rows,
                                 uint32_t cols, int* flag, cudaStream_t s);
cudaError_t launch_softmax_five_pass(const float* src, float* dst,
                                     uint32_t rows, uint32_t cols,
                                     float* scratch, int* flag,
                                     cudaStream_t s);

// --- conv.cu / gemm.cu ---------------------------------------------------
struct ConvArgs {
  const float* src;
  const float* filters;
  float* dst;
  uint32_t n, ci, h, w;
  uint32_t co, fh, fw, stride, pad;
  uint32_t ho, wo;
  int layout;  // LCNN_CHWN or LCNN_NCHW
  int precision;
  void* workspace;
  // caller-owned 64-bit sync word (zero before first use, reserved for
  // launches of one call site that never overlap): stream-K output regions
  // are zeroed inside the kernel instead of by a zero2d launch (nullptr: launch)
  unsigned long long* zsync = nullptr;
  // LCNN_CONV_IN_HWCN32 / LCNN_CONV_OUT_HWCN32: the input / output activation
  // is in the blocked [N/32][H][W][C][32] layout (run_network-internal, between
  // a ROW row-pair producer and a TAPS row-pair consumer)
  uint32_t blk = 0;
};
// 1 when the route of `a` (and the fused pool when pwin != 0) reads / writes
// the blocked layout the flags name
bool conv_hwcn32_ok(const ConvArgs& a, uint32_t pwin, uint32_t pstride);
cudaError_t launch_conv(const ConvArgs& a, cudaStream_t s);
cudaError_t launch_conv_oracle(const ConvArgs& a, uint64_t sn, uint64_t sc, uint64_t sh,
                               uint64_t sw, cudaStream_t s);
cudaError_t launch_im2col(const ConvArgs& a, cudaStream_t s);
// Workspace of the one-shot launch_conv (packed filters + run workspace).
size_t conv_workspace_bytes(const ConvArgs& a);
// Filter pre-packing: bytes of the packed operand image of a's route, the
// pack itself (a.filters -> packed), and the launch on packed filters
// (a.workspace: the run workspace, conv_workspace_bytes - conv_packed_bytes).
size_t conv_packed_bytes(const ConvArgs& a);
cudaError_t launch_conv_pack(const ConvArgs& a, void* packed, cudaStream_t s);
cudaError_t launch_conv_packed(const ConvArgs& a, const void* packed, cudaStream_t s);
// Convolution followed by a max pooling (window pwin, stride pstride) in one
// kernel; a.dst receives the POOLED output.  The packed filters are the
// layer's lcnn_conv_pack image.
bool conv_maxpool_fusable(const ConvArgs& a, uint32_t pwin, uint32_t pstride);
cudaError_t launch_conv_maxpool_packed(const ConvArgs& a, const void* packed, uint32_t pwin,
                                       uint32_t pstride, cudaStream_t s);
bool tc_gemm_supported(uint64_t m, uint64_t n, uint64_t k, const void* a,
                       const void* b);
size_t gemm_workspace_bytes(uint64_t m, uint64_t n, uint64_t k, int precision);
// fc on pre-packed weights (W^T, K-major); a_mn: x is [k][m] (CHWN producer)
size_t fc_packed_bytes(uint64_t k, uint64_t n, int precision);
size_t fc_workspace_bytes(uint64_t m, uint64_t k, int precision);
bool fc_tc_supported(uint64_t m, uint64_t n, uint64_t k, bool a_mn);
// zero a region of rows x width 32-bit words, row pitch in words (PDL kernel)
cudaError_t launch_zero2d(void* p, uint64_t pitch_words, uint64_t width_words, uint64_t rows,
                          cudaStream_t s);
cudaError_t launch_fc_pack(const float* w, uint64_t k, uint64_t n, int precision, void* packed,
                           cudaStream_t s);
// zsync: as ConvArgs::zsync (nullptr: the stream-K output is zeroed by a
// zero2d launch ahead of the kernel)
// next_packed / next_bytes: the next fc layer's packed weights, prefetched
// into L2 by each CTA once its own loads are issued (nullptr: none)
cudaError_t launch_fc_packed(const float* x, bool a_mn, const void* packed, float* c, uint64_t m,
                             uint64_t n, uint64_t k, int precision, void* ws, cudaStream_t s,
                             unsigned long long* zsync = nullptr,
                             const void* next_packed = nullptr, uint64_t next_bytes = 0);
cudaError_t launch_gemm_tc(const float* a, const float* b, float* c, uint64_t m,
                           uint64_t n, uint64_t k, int precision, void* ws,
                           cudaStream_t s);
cudaError_t launch_gemm_fp32(const float* a, const float* b, float* c, uint64_t m,
                             uint64_t n, uint64_t k, cudaStream_t s);

}  // namespace lcnn_impl
