// Softmax classifier and fully-connected layer (drop-in for the reference's
// softmax.hpp).  softmax_fused is one sm_100a kernel; softmax_reference keeps
// the five-kernel multi-pass structure (the paper's baseline) and, when asked,
// hands its intermediates back in the scratch struct.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "lcnn/device.hpp"
#include "lcnn/tensor.hpp"

namespace lcnn {

struct SoftmaxScratch {
  std::vector<float> maxv;
  std::vector<float> midv1;
  std::vector<float> midv2;
  std::vector<float> sumv;
};

struct PassReport {
  std::uint32_t materializations = 0;
  std::uint32_t full_matrix_sweeps = 0;
};

Matrix softmax_reference(const Matrix& in, SoftmaxScratch* scratch = nullptr,
                         PassReport* report = nullptr);
std::pair<Matrix, PassReport> softmax_fused(
    const Matrix& in, std::uint32_t local_buffer_limit = 16384);
Matrix fc_forward(const Matrix& in, const Matrix& weights);

// Device-resident forms (check_finite = read the non-finite flag back and
// raise DomainError; costs one 4-byte D2H + stream sync).
DeviceMatrix softmax_fused(const DeviceMatrix& in, bool check_finite = true);
// sticky_flag (device int, used when check_finite is false): the kernel sets
// it to 1 on a non-finite input and never clears it; the caller reads it later
void softmax_fused_into(const DeviceMatrix& in, DeviceMatrix& out, bool check_finite = true,
                        int* sticky_flag = nullptr);
DeviceMatrix fc_forward(const DeviceMatrix& in, const DeviceMatrix& weights);

// fc with weights packed once (lcnn_fc_pack_weights; network layers reuse the
// same weights every forward).  pack_fc_weights returns nullptr for FP32
// precision (no packed path: fc_forward runs the reference-tolerance kernel).
// The 4D form takes the producer tensor itself: CHWN is consumed in place as
// the transposed operand (the flatten costs no transform), NCHW is already
// the row-major matrix; other layouts are transformed to NCHW first.
std::shared_ptr<DeviceBuffer> pack_fc_weights(const float* d_weights, std::uint32_t k,
                                              std::uint32_t n, int precision);
// d_sync (optional): LCNN_SYNC_BYTES of zeroed device memory owned by this
// call site (lcnn_fc_forward_packed_ex): the fc zeroes its stream-K output
// in-kernel instead of launching a zeroing kernel first.
// next_packed (optional): the next fc layer's packed weights, prefetched into
// L2 by this layer's CTAs once their own loads are issued.
DeviceMatrix fc_forward_packed(const DeviceMatrix& in, const void* d_packed, std::uint32_t n,
                               int precision, void* d_sync = nullptr,
                               const DeviceBuffer* next_packed = nullptr);
DeviceMatrix fc_forward_packed(const DeviceTensor4D& in, const void* d_packed, std::uint32_t n,
                               int precision, void* d_sync = nullptr,
                               const DeviceBuffer* next_packed = nullptr);

}  // namespace lcnn
