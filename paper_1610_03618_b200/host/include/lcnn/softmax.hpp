// Softmax classifier and fully-connected layer (drop-in for the reference's
// softmax.hpp).  softmax_fused is one sm_100a kernel; softmax_reference keeps
// the five-kernel multi-pass structure (the paper's baseline) and, when asked,
// hands its intermediates back in the scratch struct.
#pragma once

#include <cstdint>
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
DeviceMatrix fc_forward(const DeviceMatrix& in, const DeviceMatrix& weights);

}  // namespace lcnn
