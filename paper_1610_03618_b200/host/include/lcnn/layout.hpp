// Layout transformation (drop-in for the reference's layout.hpp).  CHWN and
// NCHW share the C,H,W order, so converting between them is a 2D transpose
// of the [N] x [C*H*W] view -- one shared-memory-tiled sm_100a kernel.  The
// other pairs run the generic 4D permutation kernel.
#pragma once

#include <cstdint>

#include "lcnn/device.hpp"
#include "lcnn/tensor.hpp"

namespace lcnn {

bool flattenable_pair(Layout src, Layout dst);

enum class TransformKind : std::uint8_t { Tiled2D, NaivePermute };

struct TransformPlan {
  Layout src = Layout::NCHW;
  Layout dst = Layout::NCHW;
  std::uint32_t tile = 32;   // validated: power of two in [8, 128] (a hint on the GPU)
  bool wide_copy = false;    // validated: only with N >= 64 (a hint on the GPU)
  TransformKind kind = TransformKind::Tiled2D;
};

Tensor4D transform_naive(const Tensor4D& t, Layout dst);
Tensor4D transform_tiled(const Tensor4D& t, Layout dst, const TransformPlan& plan);
TransformPlan make_plan(Layout src, Layout dst, std::uint32_t n,
                        std::uint32_t c, std::uint32_t h, std::uint32_t w);
Tensor4D transform(const Tensor4D& t, Layout dst);

// Device-resident form: stream-ordered, no host round trip.
DeviceTensor4D transform(const DeviceTensor4D& t, Layout dst);

}  // namespace lcnn
