// Convolution / fully-connected entry points (conv.hpp:17-54).
// The tcgen05 implicit-GEMM kernels land in a later milestone; until then
// these entry points report UnsupportedError instead of silently falling back.
#include <cuda_runtime.h>

#include "../../include/lcnn_cuda.h"
#include "internal.h"

extern "C" {

size_t lcnn_conv_workspace_bytes(uint32_t c_o, uint32_t c_i, uint32_t f_h, uint32_t f_w) {
  return static_cast<size_t>(c_o) * c_i * f_h * f_w * sizeof(float) * 2;
}

lcnn_status lcnn_conv_forward(const float*, const float*, float*, uint32_t, uint32_t, uint32_t,
                              uint32_t, int, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                              int, void*, size_t, void*) {
  return LCNN_EUNSUPPORTED;
}

lcnn_status lcnn_gemm(const float*, const float*, float*, uint64_t, uint64_t, uint64_t, int,
                      void*) {
  return LCNN_EUNSUPPORTED;
}

}  // extern "C"
