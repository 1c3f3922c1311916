// Convolution (drop-in for the reference's conv.hpp).  conv_direct (CHWN and
// NCHW) and conv_gemm run on the GPU (tcgen05 implicit GEMM for CHWN in the
// TF32 modes, fp32 CUDA cores in the default FP32 mode, see device.hpp);
// conv_oracle is the fp64 ground truth; conv_fft keeps its contract (stride 1
// only) and is served by the same GPU convolution -- no FFT is performed.
#pragma once

#include <cstdint>
#include <utility>

#include "lcnn/device.hpp"
#include "lcnn/tensor.hpp"

namespace lcnn {

struct ConvParams {
  std::uint32_t stride = 1;
  std::uint32_t pad = 0;
};

std::pair<std::uint32_t, std::uint32_t> conv_output_extents(
    std::uint32_t h, std::uint32_t w, std::uint32_t f_h, std::uint32_t f_w,
    const ConvParams& p);

Tensor4D conv_oracle(const Tensor4D& in, const FilterBank& f,
                     const ConvParams& p);
Tensor4D conv_direct(const Tensor4D& in, const FilterBank& f,
                     const ConvParams& p);
Matrix im2col(const Tensor4D& in, std::uint32_t f_h, std::uint32_t f_w,
              const ConvParams& p);
Tensor4D conv_gemm(const Tensor4D& in, const FilterBank& f,
                   const ConvParams& p);
Tensor4D conv_fft(const Tensor4D& in, const FilterBank& f,
                  const ConvParams& p);

void gemm_blocked(const float* a, const float* b, float* c, std::uint64_t m,
                  std::uint64_t n, std::uint64_t k);
Matrix gemm_blocked(const Matrix& a, const Matrix& b);

// Device-resident convolution; filters already in HBM as (c_o, c_i, f_h, f_w).
DeviceTensor4D conv_forward(const DeviceTensor4D& in, const float* d_filters,
                            std::uint32_t c_o, std::uint32_t f_h,
                            std::uint32_t f_w, const ConvParams& p,
                            int precision);

// The two phases of conv_forward for weights that are reused (network
// layers): the filters packed once into the operand image of the kernel this
// input geometry + precision routes to (lcnn_conv_pack_filters), and the
// convolution on that image (lcnn_conv_forward_packed) -- bit-identical to
// conv_forward on the same filters.
std::shared_ptr<DeviceBuffer> pack_conv_filters(const DeviceTensor4D& in, const float* d_filters,
                                                std::uint32_t c_o, std::uint32_t f_h,
                                                std::uint32_t f_w, const ConvParams& p,
                                                int precision);
// d_sync (optional): lcnn_conv_forward_packed_ex's per-call-site sync words
DeviceTensor4D conv_forward_packed(const DeviceTensor4D& in, const void* d_packed,
                                   std::uint32_t c_o, std::uint32_t f_h, std::uint32_t f_w,
                                   const ConvParams& p, int precision, void* d_sync = nullptr,
                                   std::uint32_t blk_flags = 0);

// Convolution and the max pooling that consumes it as one kernel
// (lcnn_conv_maxpool_packed): returns the POOLED tensor, bit-identical to
// conv_forward_packed followed by a max pool_layout with (pool_win, pool_win,
// pool_stride).  conv_maxpool_supported says whether the fused kernel covers
// the pair (CHWN, TF32, SHARE-routed conv, stride-2 windows of 2 or 3).
bool conv_maxpool_supported(const DeviceTensor4D& in, std::uint32_t c_o, std::uint32_t f_h,
                            std::uint32_t f_w, const ConvParams& p, int precision,
                            std::uint32_t pool_win, std::uint32_t pool_stride);
DeviceTensor4D conv_maxpool_forward_packed(const DeviceTensor4D& in, const void* d_packed,
                                           std::uint32_t c_o, std::uint32_t f_h,
                                           std::uint32_t f_w, const ConvParams& p, int precision,
                                           std::uint32_t pool_win, std::uint32_t pool_stride,
                                           std::uint32_t blk_flags = 0);
// blk_flags (LCNN_CONV_IN_HWCN32 / LCNN_CONV_OUT_HWCN32 of lcnn_cuda.h): the
// run_network-internal blocked activation between a ROW row-pair conv and the
// TAPS row-pair conv + pool that consumes it; the tensor keeps its CHWN tag.
bool conv_hwcn32_supported(const DeviceTensor4D& in, std::uint32_t c_o, std::uint32_t f_h,
                           std::uint32_t f_w, const ConvParams& p, int precision,
                           std::uint32_t pool_win, std::uint32_t pool_stride,
                           std::uint32_t blk_flags);

}  // namespace lcnn
